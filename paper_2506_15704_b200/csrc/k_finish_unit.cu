// k_finish_unit.cu -- the back half of a decode step for a whole
// (request, KV-head) unit: its G <= 4 query-head sessions share one K/V row
// store (GQA), so the sessions whose selection is their whole probe set
// (k >= |probe|, the common case) are finished TOGETHER over the union of
// their probe rows.  Sessions that need a Top-k (k < |probe|) run the
// per-session path (finish.cuh) inside the same CTA.
//
//   union    the G sorted probe lists -> a touched-word bitmap, per-word
//            per-session bit masks and prefix counts (shared memory); every
//            union row is staged ONCE (cp.async, K and V, 4 stages of 32
//            rows) instead of once per session
//   scores   canonical fp32 dots (devmath.sdot32, the same 8-lane FFMA2
//            chains as the per-session path) for every (row, member
//            session) pair: 8-lane group g handles session g mod G
//   attend   joint online softmax over [sinks, C2] per session at tile
//            granularity; the weights w (fp32) are split into three bf16
//            terms w = hi + mid + lo (error <= 2^-24 w) and the 3G x 32
//            weight tile times the 32 x d V tile runs on the tensor cores
//            (mma.sync m16n8k16 bf16, fp32 accumulate): the GQA group is
//            what makes softmax.V a real contraction
//   checks   per session, in parallel (256 / G threads each, emulating the
//            canonical 256-wide block sum of devmath.block_sum): finite
//            scores, u = canonical fp64 softmax of C2 -> uw, |sum u - 1|
//
// Restates engine.py:167-186 (scores, Top-k pass-through, joint softmax
// output, update weights) for G sessions at once.
#include "finish.cuh"

namespace lfps {

namespace {

using namespace fin;

constexpr int kMaxG = 4;
constexpr int kUCap = 4096;              // union rows incl. sinks held in shared memory
constexpr int kWCap = 512;               // touched 32-row words
constexpr int kMaxWords = 256;           // touched-word bitmap words: m <= 262144
constexpr int kARows = 16;               // MMA M: the 3 bf16 splits of one session + zero rows
constexpr int kAStride = kTile + 8;      // bf16 per weight-tile row (80 B: ldmatrix conflict-free)

struct UnitShared {
  FinishShared fs;                       // per-session fallback path
  int p[kMaxG], mode[kMaxG];             // mode: 0 bypassed, 1 fused, 2 top-k
  int fmask, ntopk, overflow, nw, nrows;
  int wsum[kWarps];
  uint32_t l1[kMaxWords];                // touched words
  int l1pre[kMaxWords];
  int wr[kWCap];                         // word index of rank r
  uint32_t tm[kWCap][kMaxG];             // session bit masks of word r
  uint32_t base[kWCap][kMaxG];           // session list position of word r's first bit
  int rows[kUCap];                       // union entries: sinks, then (r << 5 | bit)
  float zt[kTile][kMaxG];                // tile scores (-inf: not attended)
  float fac[kMaxG];                      // tile rescale factors
  float mrun[kMaxG], srun[kMaxG];        // running max / sum (written by warp 0)
  int bad;
  double vred[kMaxG][8];                 // canonical sums: virtual-warp partials
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t* r) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Segmented OR over a warp whose lanes hold non-decreasing keys: the first
// lane of each run of equal keys returns true with the run's OR in `val`.
__device__ __forceinline__ bool seg_or(int key, uint32_t& val, bool valid) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_down_sync(LFPS_FULL, val, o);
    const int ky = __shfl_down_sync(LFPS_FULL, key, o);
    if (lane + o < 32 && ky == key) val |= y;
  }
  const int kp = __shfl_up_sync(LFPS_FULL, key, 1);
  return valid && (lane == 0 || kp != key);
}

// exclusive scan over the 256 threads (all must call)
__device__ __forceinline__ int scan_all(int v, int* wsum, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(LFPS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[warp] = x;
  __syncthreads();
  int before = 0, all = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    before += k < warp ? wsum[k] : 0;
    all += wsum[k];
  }
  __syncthreads();
  *total = all;
  return before + x - v;
}

// Canonical 256-wide block sum (devmath.block_sum) of session g's values,
// computed by the T = 256 / G threads t of group g: virtual thread
// v = t + T k holds acc[k]; virtual warp (t >> 5) + (T / 32) k.
template <int G>
__device__ __forceinline__ double group_canon_sum(const double* acc, int g, int t,
                                                  double (*vred)[8]) {
  constexpr int T = 256 / G;
#pragma unroll
  for (int k = 0; k < G; ++k) {
    const double w = warp_fold(acc[k]);
    if ((t & 31) == 0) vred[g][(t >> 5) + (T / 32) * k] = w;
  }
  __syncthreads();
  double a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = vred[g][i];
#pragma unroll
  for (int h = 4; h >= 1; h >>= 1)
#pragma unroll
    for (int i = 0; i < h; ++i) a[i] = cadd(a[i], a[i + h]);
  __syncthreads();
  return a[0];
}

// bytes of the stage region: the unit pipeline's stages (padded V rows), or
// the per-session fallback's stream_rows stages if larger
__host__ __device__ constexpr size_t unit_stage_bytes(int d) {
  return (size_t)kStages * kTile * (d * 2 + d * 2 + 16) > rows_smem(d)
             ? (size_t)kStages * kTile * (d * 2 + d * 2 + 16) : rows_smem(d);
}

template <int PQ, int G>
__global__ void __launch_bounds__(kThreads, 2) lfps_finish_unit_kernel(Ctx c, const __nv_bfloat16* q) {
  extern __shared__ __align__(128) uint8_t dyn[];
  constexpr int D = PQ * 16;
  constexpr int kRowB = D * 2;
  constexpr int kVStride = kRowB + 16;                   // padded V rows (ldmatrix.trans)
  constexpr int kStageB = kTile * (kRowB + kVStride);
  // kStages x [K tile | V tile]; also the per-session fallback's stream_rows stages
  constexpr size_t kStageTot = unit_stage_bytes(D);
  uint8_t* stages = dyn;
  __nv_bfloat16* atile = reinterpret_cast<__nv_bfloat16*>(dyn + kStageTot);
  UnitShared& sh = *reinterpret_cast<UnitShared*>(dyn + kStageTot + kMaxG * kARows * kAStride * 2);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, l8 = tid & 7, grp = tid >> 3;
  const int u = blockIdx.x;
  const int b = u / c.Hkv, h = u % c.Hkv;
  const int s0 = b * c.Hq + h * G;
  const int n = c.n_ctx[b];
  const int S = c.S;
  const int m = n - S;
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  const long long tkern0 = now_clk();

  // ---- session modes -------------------------------------------------------------
  if (tid < G) {
    const int s = s0 + tid;
    const int p = c.counts[(size_t)s * CNT_N + CNT_PROBE];
    sh.p[tid] = p;
    sh.mode[tid] = c.bypass[s] ? 0 : (k >= p ? 1 : 2);
  }
  if (tid == 0) { sh.overflow = 0; sh.bad = 0; }
  __syncthreads();
  int fmask = 0, ntopk = 0, ptot = 0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    fmask |= (sh.mode[g] == 1) << g;
    ntopk += sh.mode[g] == 2;
    ptot += sh.mode[g] == 1 ? sh.p[g] : 0;
  }
  for (int g = 0; g < G; ++g) {
    if (sh.mode[g] == 0) {
      if (tid == 0) {
        int* cnt = c.counts + (size_t)(s0 + g) * CNT_N;
        cnt[CNT_K] = 0; cnt[CNT_C2] = 0; cnt[CNT_CLAMP] = 0;
      }
    }
  }
  // ---- union of the fused sessions' probe rows -------------------------------------
  const int W = (m + 31) / 32;
  const int NL1 = (W + 31) / 32;
  bool fused = fmask != 0 && NL1 <= kMaxWords;
  // the fused sessions' probe lists, staged once into the (idle) stage memory
  int* lists = reinterpret_cast<int*>(stages);
  int loff[kMaxG];
  {
    int o = 0;
#pragma unroll
    for (int g = 0; g < G; ++g) {
      loff[g] = o;
      o += ((fmask >> g) & 1) ? sh.p[g] : 0;
    }
    if ((size_t)o * 4 > (size_t)kStages * kStageB) fused = false;   // uniform
  }
  if (fused) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      if (!((fmask >> g) & 1)) continue;
      const int* pl = c.probe_idx + (size_t)(s0 + g) * c.list_cap;
      for (int j = tid; j < sh.p[g]; j += kThreads) lists[loff[g] + j] = __ldg(pl + j);
    }
    for (int i = tid; i < NL1; i += kThreads) sh.l1[i] = 0u;
    __syncthreads();
    for (int g = 0; g < G; ++g) {
      if (!((fmask >> g) & 1)) continue;
      const int* pl = lists + loff[g];
      for (int j0 = 0; j0 < sh.p[g]; j0 += kThreads) {   // warp-uniform trip count
        const int j = j0 + tid;
        const bool ok = j < sh.p[g];
        const int w = ok ? (pl[j] - S) >> 5 : 0x7fffffff;
        uint32_t bit = ok ? 1u << (w & 31) : 0u;
        if (seg_or(ok ? w >> 5 : 0x7fffffff, bit, ok)) atomicOr(&sh.l1[w >> 5], bit);
      }
    }
    __syncthreads();
    int nw;
    const uint32_t lw = tid < NL1 ? sh.l1[tid] : 0u;
    const int pre = scan_all(__popc(lw), sh.wsum, &nw);
    if (tid < NL1) sh.l1pre[tid] = pre;
    if (nw > kWCap) fused = false;                       // uniform
    if (fused) {
      int at = pre;
      for (uint32_t x = lw; x; x &= x - 1) sh.wr[at++] = tid * 32 + __ffs(x) - 1;
      for (int i = tid; i < nw * kMaxG; i += kThreads) (&sh.tm[0][0])[i] = 0u;
      __syncthreads();
      for (int g = 0; g < G; ++g) {
        if (!((fmask >> g) & 1)) continue;
        const int* pl = lists + loff[g];
        for (int j0 = 0; j0 < sh.p[g]; j0 += kThreads) {
          const int j = j0 + tid;
          const bool ok = j < sh.p[g];
          const int li = ok ? pl[j] - S : 0x7fffffff;
          const int w = li >> 5;
          uint32_t bit = ok ? 1u << (li & 31) : 0u;
          if (seg_or(ok ? w : 0x7fffffff, bit, ok)) {
            const int r = sh.l1pre[w >> 5] + __popc(sh.l1[w >> 5] & ((1u << (w & 31)) - 1u));
            atomicOr(&sh.tm[r][g], bit);
          }
        }
      }
      __syncthreads();
      // union-row prefix and per-session list positions per word
      int carry_u = 0, carry_g[kMaxG] = {};
      for (int r0 = 0; r0 < nw; r0 += kThreads) {
        const int r = r0 + tid;
        uint32_t any = 0;
        int cg[kMaxG];
#pragma unroll
        for (int g = 0; g < kMaxG; ++g) {
          const uint32_t mk = (r < nw && g < G) ? sh.tm[r][g] : 0u;
          any |= mk;
          cg[g] = __popc(mk);
        }
        int tot;
        const int upre = scan_all(__popc(any), sh.wsum, &tot);
        if (r < nw) {
          int at = S + carry_u + upre;
          for (uint32_t x = any; x; x &= x - 1, ++at)
            if (at < kUCap) sh.rows[at] = (r << 5) | (__ffs(x) - 1);
        }
        carry_u += tot;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          int tg;
          const int gpre = scan_all(cg[g], sh.wsum, &tg);
          if (r < nw) sh.base[r][g] = carry_g[g] + gpre;
          carry_g[g] += tg;
        }
      }
      if (S + carry_u > kUCap) fused = false;           // uniform: the union does not fit
      for (int i = tid; i < S; i += kThreads) sh.rows[i] = -1 - i;   // sinks
      if (tid == 0) sh.nrows = S + carry_u;
      if (tid < kMaxG) { sh.mrun[tid] = -INFINITY; sh.srun[tid] = 0.0f; sh.fac[tid] = 1.0f; }
      // weight tiles (one per session): rows >= 3 stay zero
      for (int i = tid; i < kMaxG * kARows * kAStride; i += kThreads) atile[i] = __float2bfloat16(0.0f);
      __syncthreads();
    }
  }

  if (fused) {
    const int nrows = sh.nrows;
    const long long tclk0 = now_clk();
    if ((c.flags & LFPS_FLAG_TRACE) && tid < G && ((fmask >> tid) & 1)) {
      c.trace[(size_t)(s0 + tid) * 16 + 13] = now_ns();
      c.trace[(size_t)(s0 + tid) * 16 + 11] = tclk0 - tkern0;   // union build
    }
    const __nv_bfloat16* kb = krow(c, b, h, 0);
    const __nv_bfloat16* vb = vrow(c, b, h, 0);
    // session teams: warps [WPS g, WPS g + WPS) own session g
    constexpr int WPS = kWarps / G;                      // warps per session
    constexpr int TPS = WPS * 32;                        // threads per session
    constexpr int GPS = kGroups8 / G;                    // 8-lane groups per session
    constexpr int NTW = D / 8 / WPS;                     // n-tiles (8 dims) per warp
    const int gq = warp / WPS, lw = warp % WPS;
    const int lgrp = lw * 4 + (lane >> 3);               // group within the team
    const bool gact = (fmask >> gq) & 1;
    __nv_bfloat16* at_g = atile + gq * (kARows * kAStride);
    float2 q2[PQ];
    {
      const Part<PQ> qp = ld_part<PQ>(q + (size_t)(s0 + gq) * D, l8);
#pragma unroll
      for (int t = 0; t < PQ / 2; ++t) {
        q2[2 * t] = make_float2(bf_lo(qp.a[t]), bf_lo(qp.b[t]));
        q2[2 * t + 1] = make_float2(bf_hi(qp.a[t]), bf_hi(qp.b[t]));
      }
    }
    float* c2z = c.c2_score + (size_t)(s0 + gq) * c.list_cap;
    int bad = 0;
    float mrun = -INFINITY, srun = 0.0f;                 // team lane 0 of warp lw == 0
    float acc[NTW][4];
#pragma unroll
    for (int t = 0; t < NTW; ++t)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[t][e] = 0.0f;
    auto team_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + gq), "r"(TPS) : "memory"); };

    auto row_of = [&](int e) -> int {
      const int v = sh.rows[e];
      return v < 0 ? -1 - v : S + 32 * sh.wr[v >> 5] + (v & 31);
    };
    const int ntiles = (nrows + kTile - 1) / kTile;
    // copies: 8 threads per tile row, K and V chunks; row index fetched ahead
    auto fetch = [&](int tile) {
      const int e = tile * kTile + grp;
      return (tile < ntiles && e < nrows) ? row_of(e) : -1;
    };
    auto issue = [&](int tile, int row) {
      if (tile < ntiles && row >= 0) {
        uint8_t* st = stages + (size_t)(tile % kStages) * kStageB;
#pragma unroll
        for (int ch = l8; ch < kRowB / 16; ch += 8) {
          cp_async16(st + grp * kRowB + ch * 16,
                     reinterpret_cast<const uint8_t*>(kb + (size_t)row * D) + ch * 16);
          cp_async16(st + kTile * kRowB + grp * kVStride + ch * 16,
                     reinterpret_cast<const uint8_t*>(vb + (size_t)row * D) + ch * 16);
        }
      }
      cp_async_commit();
    };
#pragma unroll 1
    for (int t = 0; t < kStages - 1; ++t) issue(t, fetch(t));
    int ahead = fetch(kStages - 1);
#pragma unroll 1
    for (int tile = 0; tile < ntiles; ++tile) {
      cp_async_wait<kStages - 2>();
      __syncthreads();                                   // tile landed; stage tile-1 free
      issue(tile + kStages - 1, ahead);
      ahead = fetch(tile + kStages);
      if (!gact) continue;                               // whole team
      const uint8_t* st = stages + (size_t)(tile % kStages) * kStageB;
      // ---- scores: team group lgrp, tile rows lgrp + GPS i (G independent chains) ----
      {
        float pz[G];
        int vv[G];
        bool mem[G];
#pragma unroll
        for (int i = 0; i < G; ++i) {
          const int tr = lgrp + GPS * i;
          const int e = tile * kTile + tr;
          vv[i] = e < nrows ? sh.rows[e] : 0;
          mem[i] = e < nrows && (vv[i] < 0 || ((sh.tm[vv[i] >> 5][gq] >> (vv[i] & 31)) & 1u));
          const Part<PQ> kp = ld_part<PQ>(reinterpret_cast<const __nv_bfloat16*>(st + tr * kRowB), l8);
          float2 pp = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int t = 0; t < PQ / 2; ++t) {
            pp = ffma2(make_float2(bf_lo(kp.a[t]), bf_lo(kp.b[t])), q2[2 * t], pp);
            pp = ffma2(make_float2(bf_hi(kp.a[t]), bf_hi(kp.b[t])), q2[2 * t + 1], pp);
          }
          pz[i] = __fadd_rn(pp.x, pp.y);                 // canonical fold 8 (in-lane)
        }
#pragma unroll
        for (int hh = 4; hh >= 1; hh >>= 1)
#pragma unroll
          for (int i = 0; i < G; ++i) pz[i] = __fadd_rn(pz[i], __shfl_xor_sync(LFPS_FULL, pz[i], hh));
#pragma unroll
        for (int i = 0; i < G; ++i) {
          const int tr = lgrp + GPS * i;
          float z = -INFINITY;
          if (mem[i]) {
            z = __fdiv_rn(pz[i], c.sqrt_d_f32);
            bad |= !isfinite(z);
            if (vv[i] >= 0 && l8 == 0) {
              const uint32_t mk = sh.tm[vv[i] >> 5][gq];
              c2z[sh.base[vv[i] >> 5][gq] + __popc(mk & ((1u << (vv[i] & 31)) - 1u))] = z;
            }
          }
          if (l8 == 0) sh.zt[tr][gq] = z;
        }
      }
      team_sync();
      // ---- tile softmax and the bf16-split weight rows (team warp 0, lane = row) ----
      if (lw == 0) {
        const float z = sh.zt[lane][gq];
        float tm = z;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) tm = fmaxf(tm, __shfl_xor_sync(LFPS_FULL, tm, o));
        const float mnew = fmaxf(mrun, tm);
        const float f = (mrun == -INFINITY || mnew == -INFINITY) ? 1.0f : __expf(mrun - mnew);
        const float w = (z == -INFINITY) ? 0.0f : __expf(z - mnew);
        float ws = w;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) ws += __shfl_xor_sync(LFPS_FULL, ws, o);
        const __nv_bfloat16 hi = __float2bfloat16_rn(w);
        const float r1 = w - __bfloat162float(hi);
        const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
        const __nv_bfloat16 lo = __float2bfloat16_rn(r1 - __bfloat162float(mid));
        at_g[0 * kAStride + lane] = hi;
        at_g[1 * kAStride + lane] = mid;
        at_g[2 * kAStride + lane] = lo;
        mrun = mnew;
        srun = srun * f + ws;
        if (lane == 0) sh.fac[gq] = f;
      }
      team_sync();
      // ---- acc (rows hi/mid/lo) = acc * f + A (3 x 32) . V tile, on the tensor cores ----
      {
        const float f = sh.fac[gq];
#pragma unroll
        for (int t = 0; t < NTW; ++t)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[t][e] *= f;
        const uint8_t* vt = st + kTile * kRowB;
#pragma unroll
        for (int ks = 0; ks < kTile / 16; ++ks) {
          uint32_t af[4];
          {
            const int arow = (lane & 7) + ((lane >> 3) & 1) * 8;
            const int acol = ks * 16 + (lane >> 4) * 8;
            ldsm_x4(smem_addr(at_g + arow * kAStride + acol), af);
          }
#pragma unroll
          for (int t = 0; t < NTW; t += 2) {
            const int n0 = (lw * NTW + t) * 8;
            const int vrow_ = ks * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
            const int vcol = n0 + (lane >> 4) * 8;
            uint32_t bfr[4];
            ldsm_x4_t(smem_addr(vt + vrow_ * kVStride + vcol * 2), bfr);
            mma_bf16(acc[t], af, bfr[0], bfr[1]);
            mma_bf16(acc[t + 1], af, bfr[2], bfr[3]);
          }
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
    if ((c.flags & LFPS_FLAG_TRACE) && tid < G && ((fmask >> tid) & 1))
      c.trace[(size_t)(s0 + tid) * 16 + 8] = now_clk() - tclk0;
    // ---- outputs: C rows hi + mid + lo, / running sum ------------------------------
    float* cs = reinterpret_cast<float*>(stages);        // [G][3][D]
    if (gact) {
      const int a0 = lane >> 2, tq = lane & 3;
      if (a0 < 3) {
#pragma unroll
        for (int t = 0; t < NTW; ++t) {
          const int col = (lw * NTW + t) * 8 + tq * 2;
          cs[(gq * 3 + a0) * D + col] = acc[t][0];
          cs[(gq * 3 + a0) * D + col + 1] = acc[t][1];
        }
      }
      if (lw == 0 && lane == 0) sh.srun[gq] = srun;
    }
    if (bad && l8 == 0) atomicOr(&sh.bad, 1 << gq);
    __syncthreads();
    for (int i = tid; i < G * D; i += kThreads) {
      const int g = i / D, col = i % D;
      if ((fmask >> g) & 1)
        c.out[(size_t)(s0 + g) * D + col] =
            (cs[(3 * g) * D + col] + cs[(3 * g + 1) * D + col] + cs[(3 * g + 2) * D + col]) / sh.srun[g];
    }
    if ((c.flags & LFPS_FLAG_TRACE) && tid < G && ((fmask >> tid) & 1))
      c.trace[(size_t)(s0 + tid) * 16 + 9] = now_clk() - tclk0;
    // ---- per-session checks and update weights (T = 256 / G threads each) ---------------
    constexpr int T = kThreads / G;
    const int g = tid / T, t = tid % T;
    const bool act = (fmask >> g) & 1;
    const int s = s0 + g;
    const int p = sh.p[g];
    const float* z2 = c.c2_score + (size_t)s * c.list_cap;
    // max over C2 (fp32 values)
    float mf = -INFINITY;
    if (act)
      for (int j = t; j < p; j += T) mf = fmaxf(mf, z2[j]);
    for (int o = 16; o >= 1; o >>= 1) mf = fmaxf(mf, __shfl_xor_sync(LFPS_FULL, mf, o));
    float* wmax = cs + G * 3 * D;                        // [kWarps]
    if (lane == 0) wmax[warp] = mf;
    __syncthreads();
    mf = -INFINITY;
    for (int w = g * (T / 32); w < (g + 1) * (T / 32); ++w) mf = fmaxf(mf, wmax[w]);
    const double mx = (double)mf;
    // exponentials into the idle stage memory (independent, unrolled), then the
    // canonical in-order accumulation
    int eoff = 0, etot = 0;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const int pg = ((fmask >> gg) & 1) ? sh.p[gg] : 0;
      eoff += gg < g ? pg : 0;
      etot += pg;
    }
    constexpr int kEOff = 16384;                         // past the C scratch
    const bool keep = (size_t)etot * 8 <= (size_t)kStages * kStageB - kEOff;
    double* ebuf = reinterpret_cast<double*>(stages + kEOff) + eoff;
    if (keep && act) {
#pragma unroll 4
      for (int j = t; j < p; j += T) ebuf[j] = cexp(csub((double)z2[j], mx));
    }
    double accv[G];
#pragma unroll
    for (int kk = 0; kk < G; ++kk) {
      accv[kk] = 0.0;
      if (act)
        for (int j = t + T * kk; j < p; j += kCanon)
          accv[kk] = cadd(accv[kk], keep ? ebuf[j] : cexp(csub((double)z2[j], mx)));
    }
    const double tot = group_canon_sum<G>(accv, g, t, sh.vred);
    double* uw = c.uw + (size_t)s * c.list_cap;
    if (keep && act) {
#pragma unroll 4
      for (int j = t; j < p; j += T) {
        const double uu = cdiv(ebuf[j], tot);
        ebuf[j] = uu;
        uw[j] = uu;
      }
    }
#pragma unroll
    for (int kk = 0; kk < G; ++kk) {
      accv[kk] = 0.0;
      if (act)
        for (int j = t + T * kk; j < p; j += kCanon) {
          double uu;
          if (keep) {
            uu = ebuf[j];
          } else {
            uu = cdiv(cexp(csub((double)z2[j], mx)), tot);
            uw[j] = uu;
          }
          accv[kk] = cadd(accv[kk], uu);
        }
    }
    const double wsum = group_canon_sum<G>(accv, g, t, sh.vred);
    if (act) {
      int* cnt = c.counts + (size_t)s * CNT_N;
      const int* pl = c.probe_idx + (size_t)s * c.list_cap;
      int* c2i = c.c2_idx + (size_t)s * c.list_cap;
      for (int j = t; j < p; j += T) c2i[j] = __ldg(pl + j);
      if (t == 0) {
        cnt[CNT_K] = k;
        cnt[CNT_C2] = p;
        if ((sh.bad >> g) & 1) set_err(c, s, LFPS_ERR_NONFINITE_SCORES);
        else if (fabs(wsum - 1.0) > 1e-6) set_err(c, s, LFPS_ERR_WEIGHT_SUM);
        c.bw.wstat[2 * (size_t)s] = mx;
        c.bw.wstat[2 * (size_t)s + 1] = tot;
        if (c.flags & LFPS_FLAG_TRACE) {
          c.trace[(size_t)s * 16 + 10] = now_clk() - tclk0;
          c.trace[(size_t)s * 16 + 14] = now_ns();
        }
      }
    }
    __syncthreads();
  }

  // ---- sessions left to the per-session path (Top-k, or a union that does not fit) ----
  for (int g = 0; g < G; ++g) {
    const int md = sh.mode[g];
    if (md == 2 || (md == 1 && !fused)) {
      finish_session<PQ>(c, q, s0 + g, stages, sh.fs);
      __syncthreads();
    }
  }
}

}  // namespace

// G <= 4 and d in {128, 256}: the per-unit kernel; otherwise the caller uses
// the per-session kernel.  Returns cudaErrorNotSupported for other shapes.
cudaError_t launch_finish_unit(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  auto go = [&](auto kern, int pq) -> cudaError_t {
    const int d = pq * 16;
    const size_t smem = unit_stage_bytes(d) + (size_t)kMaxG * kARows * kAStride * 2 + sizeof(UnitShared);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<c.B * c.Hkv, kThreads, smem, st>>>(c, q);
    return cudaGetLastError();
  };
  if (c.d == 128) {
    switch (c.G) {
      case 1: return go(lfps_finish_unit_kernel<8, 1>, 8);
      case 2: return go(lfps_finish_unit_kernel<8, 2>, 8);
      case 4: return go(lfps_finish_unit_kernel<8, 4>, 8);
      default: return cudaErrorNotSupported;
    }
  }
  if (c.d == 256) {
    switch (c.G) {
      case 1: return go(lfps_finish_unit_kernel<16, 1>, 16);
      case 2: return go(lfps_finish_unit_kernel<16, 2>, 16);
      case 4: return go(lfps_finish_unit_kernel<16, 4>, 16);
      default: return cudaErrorNotSupported;
    }
  }
  return cudaErrorNotSupported;
}

}  // namespace lfps
