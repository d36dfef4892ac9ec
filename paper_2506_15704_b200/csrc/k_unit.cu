// k_unit.cu -- the back half of a decode step per (request, KV-head) UNIT:
// the unit's G q-head sessions over the union of their probe sets, so every
// K / V row crosses HBM -> L2 -> SM once for all G heads (the per-session
// finish, k_finish.cu, stages a row once per head).  Used when every
// non-gated head of the unit keeps its whole probe set (k >= |probe|, C2 =
// probe: the common case at 5%); a unit with a Top-k cut runs its sessions
// through finish_session (finish.cuh) inside the same launch.
//
//   slices   the context is cut into unit_nsl row ranges, one CTA each (slice
//            0 also takes the S sinks); the last CTA of a unit to finish
//            (ticket) merges the slices' softmax partials -- the split-KV
//            pattern, so small batches still fill 148 SMs
//   union    each CTA merges its range of the G heads' sorted probe lists
//            (where they start: the select kernel's slice directory) into
//            a table of rows with their member heads and list ranks, in
//            shared memory (per-head bitmaps of the range, one block scan),
//            in chunks of kChunk rows
//   rows     two rows per warp per step, both half-warps on both rows: half
//            h owns G/2 of the heads (their q, softmax states and
//            accumulators), lane l of a half canonical partial l (d/16
//            contiguous elements) of every row; each warp streams its rows
//            through its own ring of kUSt stages with cp.async (16 B per
//            lane, L2 only), warp barriers only
//   scores   z_g = (K . q_g) / fp32(sqrt d) in the canonical order of
//            devmath.sdot32 (engine.py:168-170): one fma.rn.f32.bf16 chain
//            per lane, row and head, then folds 8, 4, 2, 1 as a
//            reduce-scatter over (row, head) (each lane ends with one
//            score, one IEEE division per lane) -- bit-identical to the
//            per-session kernel; a member row's score goes to its head's C2
//            score list at its rank
//   attend   per head an online (max, sum, acc) in the base-2 domain
//            (MUFU.EX2, packed fp32x2 FMAs) over sinks u C2 (engine.py:173-181,
//            attention.py:66-85); warp states merged per CTA, slices merged
//            by the last CTA, fp32
//   checks   sinks and C2 scores finite (numerics.py:61-62); the C2 max of
//            each head to wstat for k_update.cu's canonical fp64 weights
#include "finish.cuh"

namespace lfps {

namespace {

using namespace fin;

#ifndef LFPS_UNIT_MINB
#define LFPS_UNIT_MINB 3         // resident CTAs per SM
#endif
#ifndef LFPS_UNIT_STAGES
#define LFPS_UNIT_STAGES 8
#endif
constexpr int kUSt = LFPS_UNIT_STAGES;   // ring stages per warp (one row per half-warp each)
constexpr int kChunk = 512;      // union rows per chunk (the row table in shared memory)
constexpr float kRescale = 8.0f; // log2 headroom before an online-softmax rescale

// dynamic shared memory: the row ring, at least the per-session kernel's stages
__host__ __device__ constexpr size_t unit_smem(int d) {
  return (size_t)kUSt * kWarps * 4 * d * 2 > rows_smem(d) ? (size_t)kUSt * kWarps * 4 * d * 2 : rows_smem(d);
}

template <int G>
struct UnitShared {
  int ent[kChunk + 32];                 // row | member heads << 24 (the sinks first)
  uint16_t off[(kChunk + 32) * G];      // rank of the row in each member head's list - a[g]
  int a[G], b[G];                       // the chunk's entries [a, b) of each head's list
  int next_l0, next_a[G];               // where the next chunk starts (more rows than kChunk)
  int p[G], byp[G];
  int scan[kWarps][G + 1];
  float m[kWarps][G], s[kWarps][G], mx[kWarps][G], ck[kWarps][G];
  int last;
};

template <int PQ>
__device__ __forceinline__ void lds_part(uint32_t addr, uint32_t (&w)[PQ / 2]) {
  if constexpr (PQ == 8) {
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]) : "r"(addr));
  } else {
    static_assert(PQ == 4, "d = 64 or 128");
    asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(w[0]), "=r"(w[1]) : "r"(addr));
  }
}

// Canonical folds 8, 4, 2, 1 of a half-warp's partials of two rows x HPL
// heads as a reduce-scatter: lane l16 ends with row (l16 >> 3) of head
// ((l16 >> 2) & 1 when HPL = 2).  Every add is x_l + x_(l^h) of
// devmath.sdot32's tree (IEEE addition commutes).
template <int HPL>
__device__ __forceinline__ float fold_rows(const float (&x)[2][HPL], int l16) {
  const bool b3 = (l16 & 8) != 0;
  float v;
  if constexpr (HPL == 2) {
    const bool b2 = (l16 & 4) != 0;
    const float r0 = __shfl_xor_sync(LFPS_FULL, b3 ? x[0][0] : x[1][0], 8);
    const float r1 = __shfl_xor_sync(LFPS_FULL, b3 ? x[0][1] : x[1][1], 8);
    const float a0 = __fadd_rn(b3 ? x[1][0] : x[0][0], r0);
    const float a1 = __fadd_rn(b3 ? x[1][1] : x[0][1], r1);
    v = __fadd_rn(b2 ? a1 : a0, __shfl_xor_sync(LFPS_FULL, b2 ? a0 : a1, 4));
  } else {
    static_assert(HPL == 1, "G = 2 or 4");
    v = __fadd_rn(b3 ? x[1][0] : x[0][0], __shfl_xor_sync(LFPS_FULL, b3 ? x[0][0] : x[1][0], 8));
    v = __fadd_rn(v, __shfl_xor_sync(LFPS_FULL, v, 4));
  }
  v = __fadd_rn(v, __shfl_xor_sync(LFPS_FULL, v, 2));
  v = __fadd_rn(v, __shfl_xor_sync(LFPS_FULL, v, 1));
  return v;
}

template <int PQ, int G, int RM>
__global__ void __launch_bounds__(kThreads, LFPS_UNIT_MINB)
    lfps_unit_finish_kernel(Ctx c, const __nv_bfloat16* q) {
  extern __shared__ __align__(128) uint8_t stages[];
  __shared__ FinishShared sh;
  __shared__ UnitShared<G> us;
  constexpr int D = PQ * 16;
  constexpr int kRowB = D * 2;                  // bytes of one K (or V) row
  constexpr int kStB = 4 * kRowB;               // one stage of a warp: 2 rows x (K | V)
  const int nsl = c.unit_nsl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pdl_wait();                                   // the select kernel's lists and directory
  const int ul = blockIdx.x / nsl, sl = blockIdx.x - ul * nsl;
  const int u = c.s_off / G + ul;
  const int b = u / c.Hkv, h = u - b * c.Hkv;
  const int n = c.n_ctx[b];
  const int S = c.S, m_ = n - S;
  if (tid < G) {
    const int sg = u * G + tid;
    const int* dir = c.unit_dir + (size_t)sg * (kUnitMaxSlices + 1);
    us.p[tid] = c.counts[(size_t)sg * CNT_N + CNT_PROBE];
    us.byp[tid] = c.bypass[sg];
    us.a[tid] = dir[sl];
    us.b[tid] = dir[sl + 1];
  }
  __syncthreads();
  const int k = (int)rint(c.frac * (double)n) < 1 ? 1 : (int)rint(c.frac * (double)n);
  int hmask = 0;
  bool fused = true;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (us.byp[g]) continue;
    hmask |= 1 << g;
    fused &= k >= us.p[g];
  }
  if (!fused) {                                 // a Top-k cut: the sessions one by one
    if (sl < G) finish_session<PQ, RM>(c, q, u * G + sl, stages, sh);
    pdl_trigger();
    return;
  }
  if (!hmask) {                                 // every head gated
    pdl_trigger();
    return;
  }
  // Both half-warps work on the warp's two rows of a step; half hw owns
  // heads hw HPL .. hw HPL + HPL - 1 (their q partials, softmax states and
  // accumulators), lane l16 canonical partial l16 of every row.
  constexpr int HPL = G / 2;
  const int hw = lane >> 4, l16 = lane & 15;
  const int rr = l16 >> 3;                      // the row of this lane's folded score
  const int hh = hw * HPL + (HPL == 2 ? (l16 >> 2) & 1 : 0);   // ... and its head
  const bool writer = (l16 & (8 / HPL - 1)) == 0;
  float* c2z = c.c2_score + (size_t)(u * G + hh) * c.list_cap;
  const RowMapT<RM> rmap(c, b, h);
  // copies: half hw stages row hw of a step; this lane's 16-byte chunks
  const uint8_t* ksrc = reinterpret_cast<const uint8_t*>(RM == 0 ? krow(c, b, h, 0) : c.K);
  const uint8_t* vsrc = reinterpret_cast<const uint8_t*>(RM == 0 ? vrow(c, b, h, 0) : c.V);
  uint32_t dst0 = smem_u32(stages) + warp * (kUSt * kStB) + hw * (2 * kRowB);
  if constexpr (kRowB == 256) {                 // d = 128: K chunk l16 and V chunk l16
    ksrc += l16 * 16;
    vsrc += l16 * 16;
    dst0 += l16 * 16;
  } else {                                      // d = 64: lanes 0-7 K, 8-15 V
    const int ch = l16 & 7;
    ksrc = (l16 < 8 ? ksrc : vsrc) + ch * 16;
    dst0 += (l16 < 8 ? 0 : kRowB) + ch * 16;
  }
  const uint32_t rd0 = smem_u32(stages) + warp * (kUSt * kStB) + l16 * (PQ * 2);

  // q: lane l16 holds canonical partial l16 (PQ elements, packed bf16) of its heads
  uint32_t qw[HPL][PQ / 2];
#pragma unroll
  for (int j = 0; j < HPL; ++j) {
    const uint32_t* qp =
        reinterpret_cast<const uint32_t*>(q + (size_t)(u * G + hw * HPL + j) * D) + l16 * (PQ / 2);
    if constexpr (PQ == 8) {
      const uint4 x = *reinterpret_cast<const uint4*>(qp);
      qw[j][0] = x.x; qw[j][1] = x.y; qw[j][2] = x.z; qw[j][3] = x.w;
    } else {
      const uint2 x = *reinterpret_cast<const uint2*>(qp);
      qw[j][0] = x.x; qw[j][1] = x.y;
    }
  }

  float m[HPL], ssum[HPL];
  float2 acc[HPL][PQ / 2];
#pragma unroll
  for (int j = 0; j < HPL; ++j) {
    m[j] = -INFINITY;
    ssum[j] = 0.0f;
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t) acc[j][t] = make_float2(0.0f, 0.0f);
  }
  float chk = 0.0f, mxc = -INFINITY;            // of head hh over the rows of parity rr

  // the slice's logical rows [l0, l1); chunks of <= kChunk union rows
  const int R = (m_ + nsl - 1) / nsl;
  int l0 = min(m_, sl * R);
  const int l1 = min(m_, l0 + R);
#pragma unroll 1
  for (int first = 1;; first = 0) {
    // ---- the chunk's row table: per-head bitmaps of [l0, l1) from the lists ----------
    // rows [l0, l1c): as many as the scratch (the unused ring) holds bitmaps
    // and word prefixes of
    constexpr int kScratchW = (int)(unit_smem(D) / 4 / (2 * G + 1));
    const int l1c = min(l1, l0 + kScratchW * 32);
    const int NW = (l1c - l0 + 31) >> 5;
    uint32_t* bm = reinterpret_cast<uint32_t*>(stages);           // [G][NW] (ring unused yet)
    for (int w = tid; w < G * NW; w += kThreads) bm[w] = 0u;
    __syncthreads();
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!((hmask >> g) & 1)) continue;
      const int* lg = c.probe_idx + (size_t)(u * G + g) * c.list_cap;
      const int a = us.a[g], e = us.b[g];
      for (int i0 = a + tid; i0 < e; i0 += 4 * kThreads) {
        int r[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) r[x] = i0 + x * kThreads < e ? __ldg(lg + i0 + x * kThreads) : -1;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          if (r[x] < 0) continue;
          const int o = r[x] - S - l0;
          if (o < l1c - l0) atomicOr(bm + g * NW + (o >> 5), 1u << (o & 31));
        }
      }
    }
    __syncthreads();
    const int wpt = (NW + kThreads - 1) / kThreads;
    const int w0 = min(NW, tid * wpt), w1 = min(NW, w0 + wpt);
    int v[G + 1];
#pragma unroll
    for (int i = 0; i <= G; ++i) v[i] = 0;
    for (int w = w0; w < w1; ++w) {
      uint32_t uo = 0u;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const uint32_t x = bm[g * NW + w];
        uo |= x;
        v[1 + g] += __popc(x);
      }
      v[0] += __popc(uo);
    }
    int tot0, totg[G];
    {                                           // exclusive block scans of the G + 1 counts
      int x[G + 1];
#pragma unroll
      for (int i = 0; i <= G; ++i) x[i] = v[i];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int i = 0; i <= G; ++i) {
          const int y = __shfl_up_sync(LFPS_FULL, x[i], o);
          if (lane >= o) x[i] += y;
        }
      }
      if (lane == 31) {
#pragma unroll
        for (int i = 0; i <= G; ++i) us.scan[warp][i] = x[i];
      }
      __syncthreads();
      tot0 = 0;
#pragma unroll
      for (int i = 0; i <= G; ++i) {
        int before = 0, all = 0;
#pragma unroll
        for (int k2 = 0; k2 < kWarps; ++k2) {
          const int t = us.scan[k2][i];
          before += k2 < warp ? t : 0;
          all += t;
        }
        v[i] = before + x[i] - v[i];
        if (i == 0) tot0 = all;
        else totg[i - 1] = all;
      }
    }
    const int ns = (first && sl == 0) ? S : 0;  // the sinks lead slice 0's first chunk
    // word prefixes (union, then each head) behind the bitmaps; the entries
    // are then emitted evenly over the threads (a dense band of words would
    // otherwise serialise on the thread that owns it)
    int* pre = reinterpret_cast<int*>(bm + G * NW);                // [G + 1][NW]
    {
      int run[G + 1];
#pragma unroll
      for (int i = 0; i <= G; ++i) run[i] = v[i];
      for (int w = w0; w < w1; ++w) {
        uint32_t uo = 0u;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const uint32_t x = bm[g * NW + w];
          uo |= x;
          pre[(1 + g) * NW + w] = run[1 + g];
          run[1 + g] += __popc(x);
        }
        pre[w] = run[0];
        run[0] += __popc(uo);
      }
    }
    __syncthreads();
    const int E = min(tot0, kChunk + 1);        // entry kChunk: where the next chunk starts
    for (int e = tid; e < E; e += kThreads) {
      int lo = 0, hi = NW - 1;                  // the last word with pre[w] <= e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= e) lo = mid; else hi = mid - 1;
      }
      const int w = lo;
      uint32_t x[G], uo = 0u;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        x[g] = bm[g * NW + w];
        uo |= x[g];
      }
      const int bit = __fns(uo, 0, e - pre[w] + 1);
      const uint32_t below = (1u << bit) - 1u;
      if (e < kChunk) {
        int mk = 0;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          mk |= (int)((x[g] >> bit) & 1u) << g;
          us.off[(ns + e) * G + g] = (uint16_t)(pre[(1 + g) * NW + w] + __popc(x[g] & below));
        }
        us.ent[ns + e] = (S + l0 + w * 32 + bit) | (mk << 24);
      } else {                                  // the first row of the next chunk
        us.next_l0 = l0 + w * 32 + bit;
#pragma unroll
        for (int g = 0; g < G; ++g) us.next_a[g] = us.a[g] + pre[(1 + g) * NW + w] + __popc(x[g] & below);
      }
    }
    if (tid < ns) us.ent[tid] = tid | (hmask << 24);   // sinks: every head, no rank
    const int nv = ns + min(tot0, kChunk);
    __syncthreads();                            // the table is complete; the ring may start

    // ---- the rows: 2 per warp per step, kUSt steps in flight --------------------------
    auto issue = [&](int st, int vv) {
      if (vv < nv) {
        const int row = RM == 0 ? (us.ent[vv] & 0xffffff) : rmap(us.ent[vv] & 0xffffff);
        const size_t off = (size_t)row * kRowB;
        const uint32_t dst = dst0 + st * kStB;
        cp_async16_s(dst, ksrc + off);
        if constexpr (kRowB == 256) cp_async16_s(dst + kRowB, vsrc + off);
      }
      cp_async_commit();                        // one group per step, even if empty
    };
    const int niter = (nv + 15) / 16;
#pragma unroll 1
    const int slot = warp * 2 + hw;             // the row this half-warp stages
    for (int t = 0; t < kUSt - 1; ++t) issue(t, t * 16 + slot);
    int rs = 0, ws = kUSt - 1;
#pragma unroll 1
    for (int it = 0; it < niter; ++it) {
      cp_async_wait<kUSt - 2>();                // this lane's copies of step `it` landed
      __syncwarp();                             // ... and the rest of the warp's
      issue(ws, (it + kUSt - 1) * 16 + slot);
      ws = ws + 1 == kUSt ? 0 : ws + 1;
      const uint32_t ka = rd0 + rs * kStB;       // row 0 of the step; row 1 at + 2 kRowB
      rs = rs + 1 == kUSt ? 0 : rs + 1;
      const int v0 = it * 16 + warp * 2;
      int e[2];                                 // row | member heads << 24 (no row: none)
#pragma unroll
      for (int r = 0; r < 2; ++r) e[r] = v0 + r < nv ? us.ent[v0 + r] : 0;
      float dots[2][HPL];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        uint32_t kw[PQ / 2];
        lds_part<PQ>(ka + r * 2 * kRowB, kw);
#pragma unroll
        for (int j2 = 0; j2 < HPL; ++j2) {
          float pa = 0.0f;
#pragma unroll
          for (int t = 0; t < PQ / 2; ++t) {
            pa = fma_lo(kw[t], qw[j2][t], pa);
            pa = fma_hi(kw[t], qw[j2][t], pa);
          }
          dots[r][j2] = pa;
        }
      }
      const float z = __fdiv_rn(fold_rows<HPL>(dots, l16), c.sqrt_d_f32);
      const int er = rr ? e[1] : e[0];
      if ((er >> (24 + hh)) & 1) {
        chk = __fmaf_rn(z, 0.0f, chk);
        const int vr = v0 + rr;
        if (vr >= ns) {
          mxc = fmaxf(mxc, z);
          if (writer) c2z[us.a[hh] + us.off[vr * G + hh]] = z;
        }
      }
      const float zl = z * kLog2e;
      float zg[2][HPL];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int j2 = 0; j2 < HPL; ++j2)
          zg[r][j2] = __shfl_sync(LFPS_FULL, zl, (hw << 4) + r * 8 + j2 * 4);
      const int mk0 = (e[0] >> (24 + hw * HPL)) & ((1 << HPL) - 1);   // this half's member heads
      const int mk1 = (e[1] >> (24 + hw * HPL)) & ((1 << HPL) - 1);
      if (!(mk0 | mk1)) continue;               // no row (stale stage bits) or no member
      // rescale a head only when its max grows by more than 2^kRescale (the
      // weights stay <= 2^kRescale; the state is consistent either way): one
      // rarely taken branch
      bool grow = false;
#pragma unroll
      for (int j2 = 0; j2 < HPL; ++j2)
        grow |= (((mk0 >> j2) & 1) && zg[0][j2] > m[j2] + kRescale) ||
                (((mk1 >> j2) & 1) && zg[1][j2] > m[j2] + kRescale);
      if (grow) {
#pragma unroll
        for (int j2 = 0; j2 < HPL; ++j2) {
          float mn = m[j2];
          if ((mk0 >> j2) & 1) mn = fmaxf(mn, zg[0][j2]);
          if ((mk1 >> j2) & 1) mn = fmaxf(mn, zg[1][j2]);
          if (mn > m[j2] + kRescale) {
            const float r = ex2(m[j2] - mn);
            ssum[j2] *= r;
#pragma unroll
            for (int t = 0; t < PQ / 2; ++t) acc[j2][t] = fmul2(acc[j2][t], make_float2(r, r));
            m[j2] = mn;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int mk = r ? mk1 : mk0;
        if (!mk) continue;                      // (a missing row's stage bits are stale)
        uint32_t vw[PQ / 2];
        lds_part<PQ>(ka + r * 2 * kRowB + kRowB, vw);
        float2 vf[PQ / 2];
#pragma unroll
        for (int t = 0; t < PQ / 2; ++t) vf[t] = make_float2(bf_lo(vw[t]), bf_hi(vw[t]));
#pragma unroll
        for (int j2 = 0; j2 < HPL; ++j2) {
          const float w = ((mk >> j2) & 1) ? ex2(zg[r][j2] - m[j2]) : 0.0f;
          ssum[j2] += w;
          const float2 w2 = make_float2(w, w);
#pragma unroll
          for (int t = 0; t < PQ / 2; ++t) acc[j2][t] = ffma2(vf[t], w2, acc[j2][t]);
        }
      }
    }
    cp_async_wait<0>();
    if (tot0 <= kChunk && l1c == l1) break;
    __syncthreads();                            // ring and table are free again
    if (tot0 > kChunk) {
      l0 = us.next_l0;
      if (tid < G) us.a[tid] = us.next_a[tid];
    } else {                                    // the whole range [l0, l1c) is done
      l0 = l1c;
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (tid == g) us.a[g] += totg[g];
    }
    __syncthreads();
  }
  __syncthreads();                              // the stages become merge scratch

  // ---- this CTA's 16 half-warp states -> the slice partial of each head ----------------
  float* part = reinterpret_cast<float*>(stages);   // [kWarps][G][D]
#pragma unroll
  for (int j = 0; j < HPL; ++j) {
#pragma unroll
    for (int t = 0; t < PQ / 2; ++t)
      *reinterpret_cast<float2*>(part + (warp * G + hw * HPL + j) * D + l16 * PQ + 2 * t) = acc[j][t];
  }
  if (l16 == 0) {
#pragma unroll
    for (int j = 0; j < HPL; ++j) { us.m[warp][hw * HPL + j] = m[j]; us.s[warp][hw * HPL + j] = ssum[j]; }
  }
  // the checks of head hh: rows of both parities
  mxc = fmaxf(mxc, __shfl_xor_sync(LFPS_FULL, mxc, 8));
  chk += __shfl_xor_sync(LFPS_FULL, chk, 8);
  if (writer && rr == 0) { us.mx[warp][hh] = mxc; us.ck[warp][hh] = chk; }
  __syncthreads();
  float* up = c.unit_part + ((size_t)u * kUnitMaxSlices + sl) * G * (D + 4);
  for (int x = tid; x < G * D; x += kThreads) {
    const int g = x / D, el = x - g * D;
    float M = -INFINITY;
#pragma unroll
    for (int k2 = 0; k2 < kWarps; ++k2) M = fmaxf(M, us.m[k2][g]);
    float num = 0.0f, den = 0.0f;
    if (M != -INFINITY) {
#pragma unroll 4
      for (int k2 = 0; k2 < kWarps; ++k2) {
        if (us.m[k2][g] == -INFINITY) continue;
        const float f = ex2(us.m[k2][g] - M);
        num = fmaf(f, part[(k2 * G + g) * D + el], num);
        den = fmaf(f, us.s[k2][g], den);
      }
    }
    float* pg = up + g * (D + 4);
    pg[4 + el] = num;
    if (el == 0) {
      float mx = -INFINITY, ck = 0.0f;
#pragma unroll
      for (int k2 = 0; k2 < kWarps; ++k2) { mx = fmaxf(mx, us.mx[k2][g]); ck += us.ck[k2][g]; }
      pg[0] = M;
      pg[1] = den;
      pg[2] = mx;
      pg[3] = ck;
    }
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) us.last = atomicAdd(c.unit_ticket + u, 1u) == (unsigned)(nsl - 1);
  __syncthreads();
  if (!us.last) {
    pdl_trigger();
    return;
  }
  // ---- the unit's last slice: merge the slices into every head's output -----------------
  __threadfence();
  const float* u0 = c.unit_part + (size_t)u * kUnitMaxSlices * G * (D + 4);
  for (int x = tid; x < G * D; x += kThreads) {
    const int g = x / D, el = x - g * D;
    if (!((hmask >> g) & 1)) continue;
    float M = -INFINITY;
    for (int k2 = 0; k2 < nsl; ++k2) M = fmaxf(M, __ldcg(u0 + (k2 * G + g) * (D + 4)));
    float num = 0.0f, den = 0.0f;
    for (int k2 = 0; k2 < nsl; ++k2) {
      const float* pk = u0 + (k2 * G + g) * (D + 4);
      const float mk = __ldcg(pk);
      if (mk == -INFINITY) continue;
      const float f = ex2(mk - M);
      num = fmaf(f, __ldcg(pk + 4 + el), num);
      den = fmaf(f, __ldcg(pk + 1), den);
    }
    c.out[(size_t)(u * G + g) * D + el] = num / den;
  }
  if (tid < G && ((hmask >> tid) & 1)) {
    const int s = u * G + tid;
    float mx = -INFINITY, ck = 0.0f;
    for (int k2 = 0; k2 < nsl; ++k2) {
      const float* pk = u0 + (k2 * G + tid) * (D + 4);
      mx = fmaxf(mx, __ldcg(pk + 2));
      ck += __ldcg(pk + 3);
    }
    if (!(ck == 0.0f)) set_err(c, s, LFPS_ERR_NONFINITE_SCORES);
    else c.bw.wstat[2 * (size_t)s] = (double)mx;
  }
  if (tid == 0) c.unit_ticket[u] = 0u;
  pdl_trigger();
}

template <int PQ, int G, int RM>
cudaError_t launch_unit_rm(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  const size_t smem = unit_smem(c.d);
  static DeviceOnce once;
  cudaError_t e = once.run([&] {
    cudaError_t r = cudaFuncSetAttribute(lfps_unit_finish_kernel<PQ, G, RM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(lfps_unit_finish_kernel<PQ, G, RM>,
                               cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    return r;
  });
  if (e != cudaSuccess) return e;
  const int units = c.s_cnt / G;
  return launch_pdl(lfps_unit_finish_kernel<PQ, G, RM>, dim3(units * c.unit_nsl), dim3(kThreads), smem,
                    st, c, q);
}

template <int PQ, int G>
cudaError_t launch_unit_g(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  return c.bt ? launch_unit_rm<PQ, G, 1>(c, q, st) : launch_unit_rm<PQ, G, 0>(c, q, st);
}

}  // namespace

bool unit_finish_supported(int G, int d) { return (G == 2 || G == 4) && (d == 64 || d == 128); }

// c.unit_nsl CTAs per unit, G <= unit_nsl <= kUnitMaxSlices (the
// Top-k-cut fallback needs one CTA per session)
cudaError_t launch_finish_unit(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  if (c.unit_nsl < c.G || c.unit_nsl > kUnitMaxSlices) return cudaErrorInvalidValue;
  if (c.d == 128) {
    if (c.G == 4) return launch_unit_g<8, 4>(c, q, st);
    if (c.G == 2) return launch_unit_g<8, 2>(c, q, st);
  } else if (c.d == 64) {
    if (c.G == 4) return launch_unit_g<4, 4>(c, q, st);
    if (c.G == 2) return launch_unit_g<4, 2>(c, q, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace lfps
