// k_probe.cu -- candidate construction (rest of K2): C0, C1, probe.
//
// Per session: C0 = C0_ver | C0_sla (select_initial, candidates.py:45-58);
// C1 = F & dilate(C0, offsets) where F = F_ver | F_sla is the mean filter
// and dilate sets bit j when j - delta is in C0 for some offset delta
// (expand, candidates.py:61-82, including delta = 0 being filtered);
// probe = C1 | trailing local window (finalize_probe_set,
// candidates.py:85-100).  All set algebra runs on 32-bit words; the sorted
// absolute index list is produced by an order-preserving block compaction.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t ld_or(const uint32_t* a, const uint32_t* b, int w, int W) {
  return (w >= 0 && w < W) ? (a[w] | b[w]) : 0u;
}

// bits of C0 at positions j - delta for j in word w (|delta| <= 31)
__device__ __forceinline__ uint32_t shifted(uint32_t prev, uint32_t cur, uint32_t next, int delta) {
  if (delta == 0) return cur;
  if (delta > 0) return (cur << delta) | (prev >> (32 - delta));
  const int k = -delta;
  return (cur >> k) | (next << (32 - k));
}

__global__ void __launch_bounds__(kThreads) probe_kernel(Ctx c) {
  __shared__ int scan_buf[kThreads];
  __shared__ int red[4][kThreads / 32];
  const int s = blockIdx.x;
  const int tid = threadIdx.x;
  int* cnt = c.counts + (size_t)s * CNT_N;
  if (c.bypass[s]) {
    if (tid < CNT_N) cnt[tid] = 0;
    return;
  }
  const int b = s / c.Hq;
  const int n = c.n_ctx[b];
  const int S = c.S;
  const int m = n - S;
  const int W = (m + 31) / 32;
  const uint32_t* c0v = c.bits + ((size_t)(s * 2 + 0) * 2 + 0) * c.words;
  const uint32_t* fv = c.bits + ((size_t)(s * 2 + 0) * 2 + 1) * c.words;
  const uint32_t* c0s = c.bits + ((size_t)(s * 2 + 1) * 2 + 0) * c.words;
  const uint32_t* fs = c.bits + ((size_t)(s * 2 + 1) * 2 + 1) * c.words;
  const int tail_lo = max(0, m - c.L);           // logical start of the local window

  // each thread owns a contiguous run of words
  const int per = (W + kThreads - 1) / kThreads;
  const int w0 = tid * per, w1 = min(W, w0 + per);
  int n0 = 0, n1 = 0, np = 0, nd = 0;
  // pass A: counts
  for (int w = w0; w < w1; ++w) {
    const uint32_t prev = ld_or(c0v, c0s, w - 1, W), cur = ld_or(c0v, c0s, w, W),
                   next = ld_or(c0v, c0s, w + 1, W);
    uint32_t dil = 0;
    for (int k = 0; k < c.n_off; ++k) dil |= shifted(prev, cur, next, c.off[k]);
    uint32_t valid = (w == W - 1 && (m & 31)) ? ((1u << (m & 31)) - 1u) : LFPS_FULL;
    const uint32_t c1 = (fv[w] | fs[w]) & dil & valid;
    uint32_t tail = 0;
    const int j0 = w * 32;
    if (j0 + 32 > tail_lo) {
      const int a = max(0, tail_lo - j0);
      tail = (LFPS_FULL << a) & valid;
    }
    const uint32_t pr = c1 | tail;
    n0 += __popc(cur);
    n1 += __popc(c1);
    np += __popc(pr);
    nd += __popc(cur & ~c1);
  }
  // block exclusive scan of np for the compaction offsets
  scan_buf[tid] = np;
  __syncthreads();
  for (int o = 1; o < kThreads; o <<= 1) {
    const int v = tid >= o ? scan_buf[tid - o] : 0;
    __syncthreads();
    scan_buf[tid] += v;
    __syncthreads();
  }
  int pos = scan_buf[tid] - np;
  // totals
  {
    const int lane = tid & 31, warp = tid >> 5;
    int a = n0, b2 = n1, d2 = nd;
    for (int h = 16; h >= 1; h >>= 1) {
      a += __shfl_xor_sync(LFPS_FULL, a, h);
      b2 += __shfl_xor_sync(LFPS_FULL, b2, h);
      d2 += __shfl_xor_sync(LFPS_FULL, d2, h);
    }
    if (lane == 0) { red[0][warp] = a; red[1][warp] = b2; red[2][warp] = d2; }
    __syncthreads();
    if (tid == 0) {
      int t0 = 0, t1 = 0, t3 = 0;
      for (int w = 0; w < kThreads / 32; ++w) { t0 += red[0][w]; t1 += red[1][w]; t3 += red[2][w]; }
      cnt[CNT_C0] = t0;
      cnt[CNT_C1] = t1;
      cnt[CNT_PROBE] = scan_buf[kThreads - 1];
      cnt[CNT_DROP] = t3;
    }
  }
  // pass B: emit absolute indices in ascending order
  int* out = c.probe_idx + (size_t)s * c.list_cap;
  for (int w = w0; w < w1; ++w) {
    const uint32_t prev = ld_or(c0v, c0s, w - 1, W), cur = ld_or(c0v, c0s, w, W),
                   next = ld_or(c0v, c0s, w + 1, W);
    uint32_t dil = 0;
    for (int k = 0; k < c.n_off; ++k) dil |= shifted(prev, cur, next, c.off[k]);
    uint32_t valid = (w == W - 1 && (m & 31)) ? ((1u << (m & 31)) - 1u) : LFPS_FULL;
    const uint32_t c1 = (fv[w] | fs[w]) & dil & valid;
    uint32_t tail = 0;
    const int j0 = w * 32;
    if (j0 + 32 > tail_lo) {
      const int a = max(0, tail_lo - j0);
      tail = (LFPS_FULL << a) & valid;
    }
    uint32_t pr = c1 | tail;
    while (pr) {
      const int bit = __ffs(pr) - 1;
      out[pos++] = S + j0 + bit;
      pr &= pr - 1;
    }
  }
}

}  // namespace

cudaError_t launch_probe(const Ctx& c, cudaStream_t st) {
  probe_kernel<<<c.NS, kThreads, 0, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
