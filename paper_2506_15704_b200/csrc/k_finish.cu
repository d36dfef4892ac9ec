// k_finish.cu -- the per-session back half of a decode step in ONE kernel:
// candidate scoring (K3), Top-k (K4), sparse attention (K5) and the data
// checks of the tracker update (K6; the update itself is committed by
// k_update.cu once every session has passed).  One 512-thread CTA per
// (request, q-head) session.
//
//   scores   z_j = (K[j] . q) / fp32(sqrt d) for every probe row (canonical
//            fp32 dot, devmath.sdot32; engine.py:168-170), half-warp per
//            row, 8 rows in flight per half-warp
//   top-k    k = max(1, round_half_even(frac * n)) (engine.py:167); if
//            k >= |probe| C2 = probe, else an MSB-first 4 x 8-bit radix select
//            of the k-th largest key with lowest-index ties
//            (topk_from_scores, attention.py:34-47)
//   attend   joint softmax over [sink logits, C2 logits] and sum w V
//            (engine.py:173-181): every half-warp keeps an online
//            (max, sum, acc) over its rows, 8 V rows in flight; the 32
//            partial states are merged at the end (fp32)
//   checks   sinks and C2 scores finite (softmax_weights, numerics.py:61-62,
//            called at engine.py:177 and :184); u = canonical fp64 softmax
//            of the C2 scores and |sum u - 1| <= 1e-6 (tables.py:161-163);
//            the softmax max and normaliser go to wstat for k_update.cu
#include "common.cuh"
#include "canon.cuh"
#include "frag.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kHalves = kThreads / 16;
// rows in flight per half-warp (register budget: 64 per thread at 2 CTAs/SM)
template <int PER>
constexpr int rows_in_flight() { return PER >= 16 ? 3 : (PER == 8 ? 6 : 8); }
constexpr int kCanon = 256;            // canonical block-sum width (devmath.BLOCK_THREADS)

struct FinishShared {
  float sink_z[32];
  float part_m[kHalves];
  float part_s[kHalves];
  double red[16];
  int ired[kWarps];
  unsigned hist[256];
  unsigned sel_digit;
  int sel_want;
  int warp_sums[kWarps];
};

// exclusive block scan over the 512 threads
__device__ __forceinline__ int scan512(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(LFPS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = lane < kWarps ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < kWarps; o <<= 1) {
      const int y = __shfl_up_sync(LFPS_FULL, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kWarps) warp_sums[lane] = w;
  }
  __syncthreads();
  const int before = (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
  *total = warp_sums[kWarps - 1];
  __syncthreads();
  return before;
}

// canonical 256-wide block sum (devmath.block_sum) of per-thread partials of
// threads 0..255; threads >= 256 pass 0 and are ignored; all threads get it
__device__ __forceinline__ double canon_sum(double acc, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  acc = warp_fold(acc);
  if (lane == 0 && warp < 8) red[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    double v = lane < 8 ? red[lane] : 0.0;
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1) v = cadd(v, __shfl_xor_sync(LFPS_FULL, v, h));
    if (lane == 0) red[8] = v;
  }
  __syncthreads();
  const double out = red[8];
  __syncthreads();
  return out;
}

template <int PER>
__global__ void __launch_bounds__(kThreads, 2) lfps_finish_kernel(Ctx c, const __nv_bfloat16* q) {
  constexpr int kNR = rows_in_flight<PER>();
  extern __shared__ float part_acc[];              // [kHalves][PER * 16]
  __shared__ FinishShared sh;
  const int s = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int hw = tid >> 4, hl = tid & 15;
  const int b = s / c.Hq, h = (s % c.Hq) / c.G;
  const int n = c.n_ctx[b];
  const int S = c.S;
  int* cnt = c.counts + (size_t)s * CNT_N;

  if (c.bypass[s]) {
    if (tid == 0) { cnt[CNT_K] = 0; cnt[CNT_C2] = 0; cnt[CNT_CLAMP] = 0; }
    return;
  }

  // ---- scores of the probe rows and the sinks ----------------------------------
  const int p = cnt[CNT_PROBE];
  const int* pidx = c.probe_idx + (size_t)s * c.list_cap;
  float* pz = c.probe_score + (size_t)s * c.list_cap;
  const __nv_bfloat16* kbase = krow(c, b, h, 0);
  float qf[PER];
  {
    const RawFrag<PER> qr = ld_frag<PER>(q + (size_t)s * c.d, hl);
    unpack<PER>(qr, qf);
  }
  // warp-uniform trip count: half_fold shuffles over the full warp
  for (int jw = warp * 2 * kNR; jw < p; jw += kHalves * kNR) {
    const int j0 = jw + (hw & 1) * kNR;
    RawFrag<PER> kr[kNR];
#pragma unroll
    for (int t = 0; t < kNR; ++t) {
      const int j = j0 + t;
      const int row = j < p ? __ldg(pidx + j) : 0;
      kr[t] = ld_frag<PER>(kbase + (size_t)row * c.d, hl);
    }
#pragma unroll
    for (int t = 0; t < kNR; ++t) {
      const float z = half_fold(frag_dot<PER>(kr[t], qf));
      if (hl == 0 && j0 + t < p) pz[j0 + t] = __fdiv_rn(z, c.sqrt_d_f32);
    }
  }
  if (2 * warp < S) {                      // whole warps (S may be odd)
    const RawFrag<PER> kr = ld_frag<PER>(kbase + (size_t)(hw < S ? hw : 0) * c.d, hl);
    const float z = half_fold(frag_dot<PER>(kr, qf));
    if (hl == 0 && hw < S) sh.sink_z[hw] = __fdiv_rn(z, c.sqrt_d_f32);
  }
  __syncthreads();

  // ---- Top-k ---------------------------------------------------------------------
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  int* c2i = c.c2_idx + (size_t)s * c.list_cap;
  float* c2z = c.c2_score + (size_t)s * c.list_cap;
  int k2;
  if (k >= p) {
    for (int j = tid; j < p; j += kThreads) {
      c2i[j] = pidx[j];
      c2z[j] = pz[j];
    }
    k2 = p;
  } else {
    uint32_t prefix = 0, mask = 0;
    int want = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      if (tid < 256) sh.hist[tid] = 0;
      __syncthreads();
      for (int j = tid; j < p; j += kThreads) {
        const uint32_t key = score_key(pz[j]);
        if ((key & mask) == prefix) atomicAdd(&sh.hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid < 32) {
        unsigned loc = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) loc += sh.hist[255 - 8 * tid - t];
        unsigned incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(LFPS_FULL, incl, o);
          if (tid >= o) incl += y;
        }
        const unsigned excl = incl - loc;
        if (excl < (unsigned)want && incl >= (unsigned)want) {
          unsigned cum = excl;
          for (int t = 0; t < 8; ++t) {
            const unsigned dgt = 255 - 8 * tid - t;
            const unsigned hc = sh.hist[dgt];
            if (cum + hc >= (unsigned)want) {
              sh.sel_digit = dgt;
              sh.sel_want = want - (int)cum;
              break;
            }
            cum += hc;
          }
        }
      }
      __syncthreads();
      prefix |= sh.sel_digit << shift;
      mask |= 255u << shift;
      want = sh.sel_want;
      __syncthreads();
    }
    const uint32_t kth = prefix;
    const int need_eq = want;
    int out_n = 0, eq_seen = 0;
    for (int t0 = 0; t0 < p; t0 += kThreads) {
      const int j = t0 + tid;
      const uint32_t key = j < p ? score_key(pz[j]) : 0u;
      const int gt = (j < p) && key > kth;
      const int eq = (j < p) && key == kth;
      int eq_tot, take_tot;
      const int eq_before = scan512(eq, sh.warp_sums, &eq_tot);
      const int take = gt || (eq && eq_seen + eq_before < need_eq);
      const int pos = scan512(take, sh.warp_sums, &take_tot);
      if (take) {
        c2i[out_n + pos] = pidx[j];
        c2z[out_n + pos] = pz[j];
      }
      out_n += take_tot;
      eq_seen += eq_tot;
    }
    k2 = out_n;
  }
  if (tid == 0) { cnt[CNT_K] = k; cnt[CNT_C2] = k2; }
  __syncthreads();

  // ---- attention over sinks u C2: per-half online softmax ----------------------------
  {
    float mrun = -INFINITY, srun = 0.0f;
    float acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.0f;
    const int tot = S + k2;
    for (int j0 = hw * kNR; j0 < tot; j0 += kHalves * kNR) {
      RawFrag<PER> vr[kNR];
      float zz[kNR];
#pragma unroll
      for (int t = 0; t < kNR; ++t) {
        const int j = j0 + t;
        int row = 0;
        zz[t] = -INFINITY;
        if (j < S) { row = j; zz[t] = sh.sink_z[j]; }
        else if (j < tot) { row = c2i[j - S]; zz[t] = c2z[j - S]; }   // written above
        vr[t] = ld_frag<PER>(vrow(c, b, h, row), hl);
      }
      float bm = mrun;
#pragma unroll
      for (int t = 0; t < kNR; ++t) bm = fmaxf(bm, zz[t]);
      const float rescale = mrun == -INFINITY ? 0.0f : expf(mrun - bm);
      srun *= rescale;
#pragma unroll
      for (int e = 0; e < PER; ++e) acc[e] *= rescale;
#pragma unroll
      for (int t = 0; t < kNR; ++t) {
        if (zz[t] == -INFINITY) continue;
        const float w = expf(zz[t] - bm);
        srun += w;
        float vf[PER];
        unpack<PER>(vr[t], vf);
#pragma unroll
        for (int e = 0; e < PER; ++e) acc[e] = fmaf(w, vf[e], acc[e]);
      }
      mrun = bm;
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) part_acc[hw * (PER * 16) + hl * PER + e] = acc[e];
    if (hl == 0) { sh.part_m[hw] = mrun; sh.part_s[hw] = srun; }
    __syncthreads();
    float M = -INFINITY;
#pragma unroll 4
    for (int x = 0; x < kHalves; ++x) M = fmaxf(M, sh.part_m[x]);
    float* out = c.out + (size_t)s * c.d;
    for (int t = tid; t < c.d; t += kThreads) {
      float num = 0.0f, den = 0.0f;
      for (int x = 0; x < kHalves; ++x) {
        if (sh.part_m[x] == -INFINITY) continue;
        const float f = expf(sh.part_m[x] - M);
        num = fmaf(f, part_acc[x * (PER * 16) + t], num);
        den = fmaf(f, sh.part_s[x], den);
      }
      out[t] = num / den;
    }
  }

  // ---- data checks of the update (committed by k_update.cu) ----------------------------
  int bad = 0;
  for (int j = tid; j < k2; j += kThreads) bad |= !isfinite(c2z[j]);
  if (tid < S) bad |= !isfinite(sh.sink_z[tid]);
  if (__syncthreads_or(bad)) {
    if (tid == 0) set_err(c, s, LFPS_ERR_NONFINITE_SCORES);
    return;
  }
  double mx = -INFINITY;
  for (int j = tid; j < k2; j += kThreads) mx = fmax(mx, (double)c2z[j]);
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(LFPS_FULL, mx, o));
  if (lane == 0) sh.red[warp] = mx;
  __syncthreads();
  mx = sh.red[0];
  for (int w = 1; w < kWarps; ++w) mx = fmax(mx, sh.red[w]);
  __syncthreads();
  double acc = 0.0;
  if (tid < kCanon)
    for (int j = tid; j < k2; j += kCanon) acc = cadd(acc, cexp(csub((double)c2z[j], mx)));
  const double tot = canon_sum(acc, sh.red);
  acc = 0.0;
  if (tid < kCanon)
    for (int j = tid; j < k2; j += kCanon) acc = cadd(acc, cdiv(cexp(csub((double)c2z[j], mx)), tot));
  const double wsum = canon_sum(acc, sh.red);
  if (tid == 0) {
    if (fabs(wsum - 1.0) > 1e-6) set_err(c, s, LFPS_ERR_WEIGHT_SUM);
    c.bw.wstat[2 * (size_t)s] = mx;
    c.bw.wstat[2 * (size_t)s + 1] = tot;
  }
}

template <int PER>
cudaError_t launch_finish_d(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  const size_t smem = (size_t)kHalves * PER * 16 * sizeof(float);
  lfps_finish_kernel<PER><<<c.NS, kThreads, smem, st>>>(c, q);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_finish(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  switch (c.d) {
    case 32: return launch_finish_d<2>(c, q, st);
    case 64: return launch_finish_d<4>(c, q, st);
    case 128: return launch_finish_d<8>(c, q, st);
    case 256: return launch_finish_d<16>(c, q, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
