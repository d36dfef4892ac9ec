// k_topk.cu -- per-session Top-k radix select with lower-index ties (K4).
//
// Restates topk_from_scores (attention.py:34-47) and the budget rule of
// decode_step (engine.py:167): k = max(1, round_half_even(frac * n)).  If
// k >= |probe| the whole probe set is selected; otherwise the k-th largest
// fp32 score is found by an MSB-first 4 x 8-bit radix select over
// order-preserving keys (-0.0 canonicalised to +0.0), and the selection is
// {z > kth} plus the lowest-index entries with z == kth, emitted in index
// order by an order-preserving block compaction.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// exclusive block scan of v; total returned through *total
__device__ __forceinline__ int block_excl_scan(int v, int* warp_sums, int* total) {
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
    if (lane < kWarps) warp_sums[lane] = w;   // inclusive prefix of warp totals
  }
  __syncthreads();
  const int before = (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
  *total = warp_sums[kWarps - 1];
  __syncthreads();
  return before;
}

__global__ void __launch_bounds__(kThreads) lfps_topk_kernel(Ctx c, int implicit_base) {
  __shared__ unsigned hist[256];
  __shared__ int warp_sums[kWarps];
  __shared__ unsigned sel_digit;
  __shared__ int sel_want;
  const int s = blockIdx.x, tid = threadIdx.x;
  int* cnt = c.counts + (size_t)s * CNT_N;
  if (implicit_base < 0 && c.bypass[s]) {
    if (tid == 0) { cnt[CNT_K] = 0; cnt[CNT_C2] = 0; }
    return;
  }
  const int b = s / c.Hq;
  const int n = c.n_ctx[b];
  const int p = cnt[CNT_PROBE];
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  const float* z = c.probe_score + (size_t)s * c.list_cap;
  const int* idx = c.probe_idx + (size_t)s * c.list_cap;
  int* out_i = c.c2_idx + (size_t)s * c.list_cap;
  float* out_z = c.c2_score + (size_t)s * c.list_cap;
  if (tid == 0) cnt[CNT_K] = k;
  if (k >= p) {
    for (int j = tid; j < p; j += kThreads) {
      out_i[j] = implicit_base >= 0 ? implicit_base + j : idx[j];
      out_z[j] = z[j];
    }
    if (tid == 0) cnt[CNT_C2] = p;
    return;
  }
  // ---- radix select of the k-th largest key ----
  uint32_t prefix = 0, mask = 0;
  int want = k;
  for (int shift = 24; shift >= 0; shift -= 8) {
    hist[tid] = 0;
    __syncthreads();
    for (int j = tid; j < p; j += kThreads) {
      const uint32_t key = score_key(z[j]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns digits [255 - 8 l - 7, 255 - 8 l]; suffix counts from the top
      unsigned loc = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) loc += hist[255 - 8 * tid - t];
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
          const unsigned hcount = hist[dgt];
          if (cum + hcount >= (unsigned)want) {
            sel_digit = dgt;
            sel_want = want - (int)cum;
            break;
          }
          cum += hcount;
        }
      }
    }
    __syncthreads();
    prefix |= sel_digit << shift;
    mask |= 255u << shift;
    want = sel_want;
    __syncthreads();
  }
  const uint32_t kth = prefix;
  const int need_eq = want;      // equal keys to take, lowest index first
  // ---- order-preserving compaction ----
  int base_out = 0, eq_seen = 0;
  for (int t0 = 0; t0 < p; t0 += kThreads) {
    const int j = t0 + tid;
    uint32_t key = 0;
    if (j < p) key = score_key(z[j]);
    const int gt = (j < p) && key > kth;
    const int eq = (j < p) && key == kth;
    int eq_tot;
    const int eq_before = block_excl_scan(eq, warp_sums, &eq_tot);
    const int take = gt || (eq && eq_seen + eq_before < need_eq);
    int take_tot;
    const int pos = block_excl_scan(take, warp_sums, &take_tot);
    if (take) {
      out_i[base_out + pos] = implicit_base >= 0 ? implicit_base + j : idx[j];
      out_z[base_out + pos] = z[j];
    }
    base_out += take_tot;
    eq_seen += eq_tot;
  }
  if (tid == 0) cnt[CNT_C2] = base_out;
}

}  // namespace

cudaError_t launch_topk(const Ctx& c, int implicit_base, cudaStream_t st) {
  lfps_topk_kernel<<<c.NS, kThreads, 0, st>>>(c, implicit_base);
  return cudaGetLastError();
}

}  // namespace lfps
