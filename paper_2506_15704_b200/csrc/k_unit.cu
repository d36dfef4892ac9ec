// k_unit.cu -- the back half of a decode step per (request, KV-head) UNIT
// (LFPS_FLAG_UNIT_FINISH, G = 4, d = 128): the unit's 4 q-head sessions over
// the union of their probe sets (k_union.cu), so every K / V row crosses
// HBM -> L2 -> SM -> registers ONCE for all 4 heads.  The per-session finish
// (k_finish.cu) moves each row once per head, through shared memory, with 8
// lanes per row -- it is bound by shared-memory bandwidth and issue slots
// (~34 warp instructions per session-row).  Here:
//
//   items    one 128-thread CTA (4 warps) per (unit, slice): the union
//            entries split evenly into unit_nsl slices (the unit's last
//            CTA to finish merges the slices' softmax partials: split-KV);
//            3 CTAs per SM
//   steps    a warp takes 8 union rows per step; lane (h, r) = (lane / 8,
//            lane % 8) scores row r for head h.  Rows stream through a
//            per-warp ring of kUSt steps with cp.async (16 B per lane,
//            coalesced: lanes 0-15 one row, 16-31 the next), padded to 272
//            bytes per row so that the 8 lanes of one shared-memory phase
//            (8 rows at one chunk offset) hit 8 distinct bank groups
//   scores   z = (K . q_h) / fp32(sqrt d) in the canonical order of
//            devmath.sdot32 (engine.py:168-170): 16 partials of 8 contiguous
//            elements, each a chain of fma.rn.f32.bf16 (the exact bf16
//            product, one rounding), folded 8, 4, 2, 1 in the lane, IEEE
//            division -- bit-identical to the per-session kernel.  q_h stays
//            in registers (64 packed words); a member row's score goes to
//            its head's C2 score list at its rank
//   attend   per head an online softmax (base 2, lazy max: it moves only
//            when a step's max exceeds it by 2^8) and sum w V on the tensor
//            cores: one mma.m16n8k8 per 16 dims and step multiplies V^T
//            (ldmatrix.trans from the staged rows) by W[8 rows x 8] whose 8
//            columns are the 4 heads' bf16 high and low weight parts (w -
//            hi, rounded: |error| <= 2^-18 w); fp32 accumulation, checked
//            against the fp64 oracle to 1e-5 relative L2
//   checks   sinks and C2 scores finite (numerics.py:61-62); each head's C2
//            max to wstat for k_update.cu's canonical fp64 weights
#include "rows.cuh"

namespace lfps {

namespace {

using namespace rows;

constexpr int kUThreads = 128;
constexpr int kUWarps = kUThreads / 32;
constexpr int kUG = 4;                   // heads per unit
constexpr int kUD = 128;                 // head dimension
#ifndef LFPS_UNIT_STAGES
#define LFPS_UNIT_STAGES 3
#endif
#ifndef LFPS_UNIT_MINB
#define LFPS_UNIT_MINB 3
#endif
constexpr int kUSt = LFPS_UNIT_STAGES;   // ring steps per warp
constexpr int kRowP = 272;               // padded shared row: 256 B + 16
constexpr int kStepB = 2 * 8 * kRowP;    // one step: 8 K rows, then 8 V rows
constexpr int kRingB = kUWarps * kUSt * kStepB;
constexpr int kEC = 1024;                // union entries per shared-memory chunk
constexpr size_t kUnitSmem = (size_t)kRingB + kEC * 20;
constexpr float kRescale = 8.0f;         // log2 headroom before an online-softmax rescale

static_assert((size_t)kUWarps * kUG * kUD * 4 <= kUnitSmem, "merge scratch fits the ring");

struct UnitShared {
  float m[kUWarps][kUG], s[kUWarps][kUG], mx[kUWarps][kUG], ck[kUWarps][kUG];
  int hmask, last;
};

__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                          uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
// D[16 x 8] += A[16 x 8] B[8 x 8], bf16 in, fp32 accumulate
__device__ __forceinline__ void mma_k8(float* d, uint32_t a0, uint32_t a1, uint32_t b) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
               "{%0, %1, %2, %3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3]) : "r"(a0), "r"(a1), "r"(b));
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

template <int RM>
__global__ void __launch_bounds__(kUThreads, LFPS_UNIT_MINB) lfps_unit_finish_kernel(Ctx c, const __nv_bfloat16* q) {
  extern __shared__ __align__(128) uint8_t ring[];
  __shared__ UnitShared us;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nsl = c.unit_nsl;
  pdl_wait();                                   // the union kernel's table
  const int ul = blockIdx.x / nsl, sl = blockIdx.x - ul * nsl;
  const int u = c.s_off / kUG + ul;
  const int U = c.unit_count[u];
  if (U <= 0) {                                 // -1: a Top-k cut (per-session finish); 0: all gated
    pdl_trigger();
    return;
  }
  const int b = u / c.Hkv, hk = u - b * c.Hkv;
  if (tid == 0) {
    int hm = 0;
#pragma unroll
    for (int g = 0; g < kUG; ++g) hm |= (c.bypass[u * kUG + g] ? 0 : 1) << g;
    us.hmask = hm;
  }
  const int e0 = (int)((long long)U * sl / nsl), e1 = (int)((long long)U * (sl + 1) / nsl);
  const int h = lane >> 3, r = lane & 7;        // this lane's head and row of a step
  const int sh = u * kUG + h;
  const int* ent = c.unit_ent + (size_t)u * c.unit_cap;
  const int* rnk = c.unit_rank + (size_t)u * c.unit_cap * 4;
  float* c2z = c.c2_score + (size_t)sh * c.list_cap;

  // q of head h: canonical partial j = elements 8 j .. 8 j + 7 = words 4 j .. 4 j + 3
  uint32_t qw[64];
  {
    const uint4* qp = reinterpret_cast<const uint4*>(q + (size_t)sh * kUD);
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const uint4 x = __ldg(qp + t);
      qw[4 * t] = x.x; qw[4 * t + 1] = x.y; qw[4 * t + 2] = x.z; qw[4 * t + 3] = x.w;
    }
  }

  // ---- the entries, kEC at a time in shared memory; a warp's steps w, w + 4, ... -------
  const RowMapT<RM> rmap(c, b, hk);
  const uint8_t* kb = reinterpret_cast<const uint8_t*>(RM == 0 ? krow(c, b, hk, 0) : c.K);
  const uint8_t* vb = reinterpret_cast<const uint8_t*>(RM == 0 ? vrow(c, b, hk, 0) : c.V);
  const uint32_t wring = smem_u32(ring) + warp * (kUSt * kStepB);
  int* sent = reinterpret_cast<int*>(ring + kRingB);             // [kEC] entries
  int4* srk = reinterpret_cast<int4*>(ring + kRingB + kEC * 4);  // [kEC] list ranks
  // stale slots of rows past the end meet the mma with weight 0: zero them once
  for (int o = lane * 16; o < kUSt * kStepB; o += 32 * 16)
    asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(wring + o), "r"(0u) : "memory");
  const int cc = lane & 15, rh = lane >> 4;     // copies: chunk cc of rows 2 i + rh

  float acc[8][4];                              // D[dims 16 x + (lane / 4) (+8)][head lane % 4, hi | lo]
#pragma unroll
  for (int x = 0; x < 8; ++x) acc[x][0] = acc[x][1] = acc[x][2] = acc[x][3] = 0.0f;
  float mo = -INFINITY, ma = -INFINITY;         // running max of head h (weights) / head lane % 4 (acc)
  float ssum = 0.0f, chk = 0.0f, mxc = -INFINITY;
  const int t4 = lane & 3, nn = lane >> 2;      // mma B fragment: rows 2 t4, 2 t4 + 1, column nn
  const int bsrc = (nn >> 1) * 8 + 2 * t4;
  const uint32_t vlane = 8 * kRowP + (lane & 7) * kRowP + (lane >> 3) * 16;

#pragma unroll 1
  for (int c0 = e0; c0 < e1; c0 += kEC) {
    const int ne = min(kEC, e1 - c0);
    __syncthreads();                            // the previous chunk's table is consumed
    for (int i = tid; i < ne; i += kUThreads) {
      sent[i] = __ldg(ent + c0 + i);
      srk[i] = __ldg(reinterpret_cast<const int4*>(rnk) + c0 + i);
    }
    __syncthreads();
    const int nsteps = (ne + 7) >> 3;
    const int nloc = nsteps > warp ? (nsteps - warp + kUWarps - 1) / kUWarps : 0;
    // copy the K and V rows of local step t into ring slot `slot`
    auto issue = [&](int slot, int t) {
      if (t < nloc) {
        const uint32_t dst = wring + slot * kStepB + cc * 16;
        const int eb = (warp + kUWarps * t) * 8;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = eb + 2 * i + rh;
          if (e >= ne) continue;
          const int r0 = sent[e] & 0xffffff;
          const int row = RM == 0 ? r0 : rmap(r0);
          const size_t off = (size_t)row * (kUD * 2) + cc * 16;
          cp_async16_s(dst + (2 * i + rh) * kRowP, kb + off);
          cp_async16_s(dst + (8 + 2 * i + rh) * kRowP, vb + off);
        }
      }
      cp_async_commit();                        // one group per step, even if empty
    };
#pragma unroll 1
    for (int t = 0; t < kUSt - 1; ++t) issue(t, t);
#pragma unroll 1
    for (int t = 0; t < nloc; ++t) {
      cp_async_wait<kUSt - 2>();                // this lane's copies of step t landed
      __syncwarp();                             // ... and the warp's; slot t - 1 is free
      issue((t + kUSt - 1) % kUSt, t + kUSt - 1);
      const uint32_t kst = wring + (t % kUSt) * kStepB;
      const int e = (warp + kUWarps * t) * 8 + r;
      const int en = e < ne ? sent[e] : 0;      // (0: no row)
      const int rk = (&srk[e < ne ? e : 0].x)[h];

      // ---- the canonical score of row r for head h -----------------------------------
      float x8[8];
      const uint32_t kr = kst + r * kRowP;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint4 kv = lds128(kr + j * 16);
        float p = 0.0f;
        p = fma_lo(kv.x, qw[4 * j], p);
        p = fma_hi(kv.x, qw[4 * j], p);
        p = fma_lo(kv.y, qw[4 * j + 1], p);
        p = fma_hi(kv.y, qw[4 * j + 1], p);
        p = fma_lo(kv.z, qw[4 * j + 2], p);
        p = fma_hi(kv.z, qw[4 * j + 2], p);
        p = fma_lo(kv.w, qw[4 * j + 3], p);
        p = fma_hi(kv.w, qw[4 * j + 3], p);
        if (j < 8) x8[j] = p;
        else x8[j - 8] = __fadd_rn(x8[j - 8], p);
      }
      const float y0 = __fadd_rn(x8[0], x8[4]), y1 = __fadd_rn(x8[1], x8[5]);
      const float y2 = __fadd_rn(x8[2], x8[6]), y3 = __fadd_rn(x8[3], x8[7]);
      const float z = __fdiv_rn(__fadd_rn(__fadd_rn(y0, y2), __fadd_rn(y1, y3)), c.sqrt_d_f32);

      const bool mem = (en >> (24 + h)) & 1;
      if (mem) {
        chk = __fmaf_rn(z, 0.0f, chk);
        if (!((en >> 28) & 1)) {                // a C2 row (not a sink)
          mxc = fmaxf(mxc, z);
          c2z[rk] = z;
        }
      }
      // ---- online softmax (lazy max) and sum w V ---------------------------------------
      const float zl = mem ? z * kLog2e : -INFINITY;
      float mh = fmaxf(zl, __shfl_xor_sync(LFPS_FULL, zl, 1));
      mh = fmaxf(mh, __shfl_xor_sync(LFPS_FULL, mh, 2));
      mh = fmaxf(mh, __shfl_xor_sync(LFPS_FULL, mh, 4));        // step max of head h
      const float ta = __shfl_sync(LFPS_FULL, mh, t4 * 8);      // ... of head lane % 4
      const bool ga = ta > ma + kRescale;
      if (__any_sync(LFPS_FULL, ga)) {
        const float f = ga ? ex2(ma - ta) : 1.0f;
#pragma unroll
        for (int x = 0; x < 8; ++x) {
          acc[x][0] *= f; acc[x][1] *= f; acc[x][2] *= f; acc[x][3] *= f;
        }
        ma = ga ? ta : ma;
      }
      if (mh > mo + kRescale) {
        ssum *= ex2(mo - mh);
        mo = mh;
      }
      const float w = mem ? ex2(zl - mo) : 0.0f;
      ssum += w;
      // W column 2 h' + 0 / 1 = head h' high / low parts; lane 8 h' + 2 i holds
      // rows 2 i, 2 i + 1 of head h' packed
      const float wn = __shfl_xor_sync(LFPS_FULL, w, 1);
      const float wa = (r & 1) ? wn : w, wb = (r & 1) ? w : wn;
      const uint32_t hi = cvt_bf16x2(wa, wb);
      const uint32_t lo = cvt_bf16x2(wa - bf_lo(hi), wb - bf_hi(hi));
      const uint32_t bh = __shfl_sync(LFPS_FULL, hi, bsrc);
      const uint32_t bl = __shfl_sync(LFPS_FULL, lo, bsrc);
      const uint32_t bw = (nn & 1) ? bl : bh;
      const uint32_t vr = kst + vlane;
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(vr + x * 64, a0, a1, a2, a3); // dims 32 x .. 32 x + 31 of the 8 rows
        mma_k8(acc[2 * x], a0, a1, bw);
        mma_k8(acc[2 * x + 1], a2, a3, bw);
      }
    }
    cp_async_wait<0>();
  }
  cp_async_wait<0>();
  __syncthreads();                              // the ring becomes merge scratch

  // ---- this CTA's 4 warp states -> the slice partial of each head ------------------------
  float* part = reinterpret_cast<float*>(ring);   // [kUWarps][kUG][kUD]
#pragma unroll
  for (int x = 0; x < 8; ++x) {
    part[(warp * kUG + t4) * kUD + 16 * x + nn] = acc[x][0] + acc[x][1];
    part[(warp * kUG + t4) * kUD + 16 * x + 8 + nn] = acc[x][2] + acc[x][3];
  }
#pragma unroll
  for (int o = 1; o <= 4; o <<= 1) {
    ssum += __shfl_xor_sync(LFPS_FULL, ssum, o);
    chk += __shfl_xor_sync(LFPS_FULL, chk, o);
    mxc = fmaxf(mxc, __shfl_xor_sync(LFPS_FULL, mxc, o));
  }
  if (r == 0) {
    us.m[warp][h] = mo;
    us.s[warp][h] = ssum;
    us.mx[warp][h] = mxc;
    us.ck[warp][h] = chk;
  }
  __syncthreads();
  const int hmask = us.hmask;
  float* up = c.unit_part + ((size_t)u * kUnitMaxSlices + sl) * kUG * (kUD + 4);
  for (int x = tid; x < kUG * kUD; x += kUThreads) {
    const int g = x / kUD, el = x - g * kUD;
    float M = -INFINITY;
#pragma unroll
    for (int k2 = 0; k2 < kUWarps; ++k2) M = fmaxf(M, us.m[k2][g]);
    float num = 0.0f, den = 0.0f;
    if (M != -INFINITY) {
#pragma unroll
      for (int k2 = 0; k2 < kUWarps; ++k2) {
        if (us.m[k2][g] == -INFINITY) continue;
        const float f = ex2(us.m[k2][g] - M);
        num = fmaf(f, part[(k2 * kUG + g) * kUD + el], num);
        den = fmaf(f, us.s[k2][g], den);
      }
    }
    float* pg = up + g * (kUD + 4);
    pg[4 + el] = num;
    if (el == 0) {
      float mx = -INFINITY, ck = 0.0f;
#pragma unroll
      for (int k2 = 0; k2 < kUWarps; ++k2) { mx = fmaxf(mx, us.mx[k2][g]); ck += us.ck[k2][g]; }
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
  const float* u0 = c.unit_part + (size_t)u * kUnitMaxSlices * kUG * (kUD + 4);
  for (int x = tid; x < kUG * kUD; x += kUThreads) {
    const int g = x / kUD, el = x - g * kUD;
    if (!((hmask >> g) & 1)) continue;
    float M = -INFINITY;
    for (int k2 = 0; k2 < nsl; ++k2) M = fmaxf(M, __ldcg(u0 + (k2 * kUG + g) * (kUD + 4)));
    float num = 0.0f, den = 0.0f;
    for (int k2 = 0; k2 < nsl; ++k2) {
      const float* pk = u0 + (k2 * kUG + g) * (kUD + 4);
      const float mk = __ldcg(pk);
      if (mk == -INFINITY) continue;
      const float f = ex2(mk - M);
      num = fmaf(f, __ldcg(pk + 4 + el), num);
      den = fmaf(f, __ldcg(pk + 1), den);
    }
    c.out[(size_t)(u * kUG + g) * kUD + el] = num / den;
  }
  if (tid < kUG && ((hmask >> tid) & 1)) {
    const int s = u * kUG + tid;
    float mx = -INFINITY, ck = 0.0f;
    for (int k2 = 0; k2 < nsl; ++k2) {
      const float* pk = u0 + (k2 * kUG + tid) * (kUD + 4);
      mx = fmaxf(mx, __ldcg(pk + 2));
      ck += __ldcg(pk + 3);
    }
    if (!(ck == 0.0f)) set_err(c, s, LFPS_ERR_NONFINITE_SCORES);
    else c.bw.wstat[2 * (size_t)s] = (double)mx;
  }
  if (tid == 0) c.unit_ticket[u] = 0u;
  pdl_trigger();
}

template <int RM>
cudaError_t launch_unit_rm(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  static DeviceOnce once;
  cudaError_t e = once.run([&] {
    cudaError_t r = cudaFuncSetAttribute(lfps_unit_finish_kernel<RM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kUnitSmem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(lfps_unit_finish_kernel<RM>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    return r;
  });
  if (e != cudaSuccess) return e;
  const int units = c.s_cnt / kUG;
  return launch_pdl(lfps_unit_finish_kernel<RM>, dim3(units * c.unit_nsl), dim3(kUThreads), kUnitSmem, st,
                    c, q);
}

}  // namespace

bool unit_finish_supported(int G, int d) { return G == kUG && d == kUD; }

// c.unit_nsl CTAs per unit, 1 <= unit_nsl <= kUnitMaxSlices
cudaError_t launch_finish_unit(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  if (c.unit_nsl < 1 || c.unit_nsl > kUnitMaxSlices || !unit_finish_supported(c.G, c.d))
    return cudaErrorInvalidValue;
  return c.bt ? launch_unit_rm<1>(c, q, st) : launch_unit_rm<0>(c, q, st);
}

}  // namespace lfps
