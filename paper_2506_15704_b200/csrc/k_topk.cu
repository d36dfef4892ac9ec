// k_topk.cu -- exact-path Top-k over every non-sink score of a session (KX).
//
// Restates topk_from_scores (attention.py:34-47) applied to the full score
// vector of exact_topk_step (bench.py:73-80), with the budget rule of
// decode_step (engine.py:167): k = max(1, round_half_even(frac * n)).  If
// k >= m every non-sink row is selected; otherwise the selection is
// {z > kth} plus the lowest-index entries with z == kth, emitted in index
// order.  Keys are order-preserving uint32 maps of the fp32 scores with -0.0
// canonicalised to +0.0 (canon.cuh score_key).  One 512-thread CTA per
// session, three streaming passes over its m scores:
//
//   1  2048-bin histogram of the top 11 key bits (shared-memory atomics)
//      -> the bin holding the k-th largest key, and how many keys lie above;
//   2  that bin's (key, index) pairs are collected (shared memory, or the
//      session's uw scratch when they do not fit), and every warp counts the
//      keys of its index chunk that lie in higher bins;
//   3  an MSB-first 3 x 7-bit radix select over the candidates gives the
//      exact k-th key; each warp then re-walks its chunk and writes its
//      selections at ballot/popc offsets, so the output is sorted.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kBins = 2048;                 // top 11 key bits
constexpr int kShift = 21;
constexpr int kSmemCand = 6144;             // candidates kept in shared memory

struct TopkShared {
  unsigned hist[kBins];
  uint2 cand[kSmemCand];                    // (key, index)
  int wsum[kWarps];
  int above[kWarps];                        // keys in higher bins, per warp chunk
  int gtc[kWarps], eqc[kWarps];             // candidates > kth / == kth, per warp chunk
  int ncand;
  int sel_bin, sel_want;
  unsigned sel_digit;
};

__global__ void __launch_bounds__(kThreads) lfps_exact_topk_kernel(Ctx c) {
  extern __shared__ uint8_t dyn[];
  TopkShared& sh = *reinterpret_cast<TopkShared*>(dyn);
  const int s = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  int* cnt = c.counts + (size_t)s * CNT_N;
  const int b = s / c.Hq;
  const int n = c.n_ctx[b];
  const int S = c.S;
  const int p = cnt[CNT_PROBE];                    // = m, set by the score kernel
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  const float* z = c.probe_score + (size_t)s * c.list_cap;
  int* out_i = c.c2_idx + (size_t)s * c.list_cap;
  float* out_z = c.c2_score + (size_t)s * c.list_cap;
  if (tid == 0) cnt[CNT_K] = k;
  if (k >= p) {
    for (int j = tid; j < p; j += kThreads) {
      out_i[j] = S + j;
      out_z[j] = z[j];
    }
    if (tid == 0) cnt[CNT_C2] = p;
    return;
  }
  // ---- pass 1: histogram of the top key bits -------------------------------------
  for (int i = tid; i < kBins; i += kThreads) sh.hist[i] = 0;
  if (tid == 0) sh.ncand = 0;
  __syncthreads();
  for (int j = tid; j < p; j += kThreads) atomicAdd(&sh.hist[score_key(z[j]) >> kShift], 1u);
  __syncthreads();
  {
    // thread t owns bins [kBins - 4 t - 4, kBins - 4 t) (descending order)
    unsigned loc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) loc += sh.hist[kBins - 1 - 4 * tid - i];
    unsigned x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(LFPS_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sh.wsum[warp] = (int)x;
    __syncthreads();
    unsigned before = 0;
    for (int w = 0; w < warp; ++w) before += (unsigned)sh.wsum[w];
    const unsigned excl = before + x - loc;
    if (excl < (unsigned)k && excl + loc >= (unsigned)k) {
      unsigned cum = excl;
      for (int i = 0; i < 4; ++i) {
        const int bin = kBins - 1 - 4 * tid - i;
        const unsigned hc = sh.hist[bin];
        if (cum + hc >= (unsigned)k) {
          sh.sel_bin = bin;
          sh.sel_want = k - (int)cum;
          break;
        }
        cum += hc;
      }
    }
    __syncthreads();
  }
  const unsigned bstar = (unsigned)sh.sel_bin;
  const int nc = (int)sh.hist[bstar];
  uint2* cand = nc <= kSmemCand ? sh.cand : reinterpret_cast<uint2*>(c.uw + (size_t)s * c.list_cap);
  // ---- pass 2: candidates of the k-th bin; keys above it per warp chunk ----------------
  const int chunk = (p + kWarps - 1) / kWarps;
  const int j0 = warp * chunk, j1 = min(p, j0 + chunk);
  int above = 0;
  for (int j = j0 + lane; j < j1; j += 32) {
    const uint32_t key = score_key(z[j]);
    const uint32_t bin = key >> kShift;
    above += bin > bstar;
    if (bin == bstar) {
      const int at = atomicAdd(&sh.ncand, 1);
      cand[at] = make_uint2(key, (uint32_t)j);
    }
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) above += __shfl_xor_sync(LFPS_FULL, above, o);
  if (lane == 0) { sh.above[warp] = above; sh.gtc[warp] = 0; sh.eqc[warp] = 0; }
  __syncthreads();
  // ---- pass 3: radix select within the bin (3 x 7 bits) -----------------------------
  uint32_t prefix = bstar << kShift, mask = ~0u << kShift;
  int want = sh.sel_want;
  for (int shift = 14; shift >= 0; shift -= 7) {
    if (tid < 128) sh.hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < nc; i += kThreads) {
      const uint32_t key = cand[i].x;
      if ((key & mask) == prefix) atomicAdd(&sh.hist[(key >> shift) & 127u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      // lane l owns digits [127 - 4 l - 3, 127 - 4 l]; suffix counts from the top
      unsigned loc = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) loc += sh.hist[127 - 4 * tid - t];
      unsigned incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(LFPS_FULL, incl, o);
        if (tid >= o) incl += y;
      }
      const unsigned excl = incl - loc;
      if (excl < (unsigned)want && incl >= (unsigned)want) {
        unsigned cum = excl;
        for (int t = 0; t < 4; ++t) {
          const unsigned dgt = 127 - 4 * tid - t;
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
    mask |= 127u << shift;
    want = sh.sel_want;
    __syncthreads();
  }
  const uint32_t kth = prefix;
  const int need_eq = want;                        // equal keys to take, lowest index first
  // per-warp-chunk counts of candidates above / equal to kth
  for (int i = tid; i < nc; i += kThreads) {
    const uint2 e = cand[i];
    const int w = (int)e.y / chunk;
    if (e.x > kth) atomicAdd(&sh.gtc[w], 1);
    else if (e.x == kth) atomicAdd(&sh.eqc[w], 1);
  }
  __syncthreads();
  // ---- ordered emission: warp w walks its chunk in index order --------------------------
  int out_at = 0, eq_at = 0;
  for (int w = 0; w < warp; ++w) {
    const int eq = sh.eqc[w];
    const int eq_take = max(0, min(eq, need_eq - eq_at));
    out_at += sh.above[w] + sh.gtc[w] + eq_take;
    eq_at += eq;
  }
  for (int base = j0; base < j1; base += 32) {
    const int j = base + lane;
    const uint32_t key = j < j1 ? score_key(z[j]) : 0u;
    const bool gt = j < j1 && key > kth;
    const bool eq = j < j1 && key == kth;
    const uint32_t eqm = __ballot_sync(LFPS_FULL, eq);
    const int my_eq = eq_at + __popc(eqm & ((1u << lane) - 1u));
    const bool take = gt || (eq && my_eq < need_eq);
    const uint32_t tm = __ballot_sync(LFPS_FULL, take);
    if (take) {
      const int pos = out_at + __popc(tm & ((1u << lane) - 1u));
      out_i[pos] = S + j;
      out_z[pos] = z[j];
    }
    out_at += __popc(tm);
    eq_at += __popc(eqm);
  }
  if (warp == kWarps - 1 && lane == 0) cnt[CNT_C2] = out_at;
}

}  // namespace

cudaError_t launch_topk(const Ctx& c, int /*implicit_base*/, cudaStream_t st) {
  static bool set = false;
  const size_t smem = sizeof(TopkShared);
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(lfps_exact_topk_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    set = true;
  }
  lfps_exact_topk_kernel<<<c.NS, kThreads, smem, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
