// k_probe.cu -- candidate construction (rest of K2): C0, C1, probe.
//
// Per session: C0 = C0_ver | C0_sla (select_initial, candidates.py:45-58);
// C1 = F & dilate(C0, offsets) where F = F_ver | F_sla is the mean filter
// and dilate sets bit j when j - delta is in C0 for some offset delta
// (expand, candidates.py:61-82, including delta = 0 being filtered);
// probe = C1 | trailing local window (finalize_probe_set,
// candidates.py:85-100).  Set algebra on 32-bit words, one word per lane
// (coalesced), neighbours through warp shuffles; the sorted absolute index
// list comes from an order-preserving two-phase compaction.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// bits of C0 at positions j - delta for j in word w (|delta| <= 31)
__device__ __forceinline__ uint32_t shifted(uint32_t prev, uint32_t cur, uint32_t next, int delta) {
  if (delta == 0) return cur;
  if (delta > 0) return (cur << delta) | (prev >> (32 - delta));
  const int k = -delta;
  return (cur >> k) | (next << (32 - k));
}

__global__ void __launch_bounds__(kThreads) probe_kernel(Ctx c) {
  extern __shared__ uint32_t pwords[];           // [W] probe words
  __shared__ int blk[192];                        // per 32-word block counts -> offsets
  __shared__ int red[4][kWarps];
  const int s = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
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
  const int nblk = (W + 31) / 32;
  const uint32_t* c0v = c.bits + ((size_t)(s * 2 + 0) * 2 + 0) * c.words;
  const uint32_t* fv = c.bits + ((size_t)(s * 2 + 0) * 2 + 1) * c.words;
  const uint32_t* c0s = c.bits + ((size_t)(s * 2 + 1) * 2 + 0) * c.words;
  const uint32_t* fs = c.bits + ((size_t)(s * 2 + 1) * 2 + 1) * c.words;
  const int tail_lo = max(0, m - c.L);           // logical start of the local window
  const uint32_t last_valid = (m & 31) ? ((1u << (m & 31)) - 1u) : LFPS_FULL;

  // phase A: probe words + counts
  int n0 = 0, n1 = 0, nd = 0;
  for (int bk = warp; bk < nblk; bk += kWarps) {
    const int w = bk * 32 + lane;
    const bool in = w < W;
    const uint32_t cur = in ? (c0v[w] | c0s[w]) : 0u;
    const uint32_t f = in ? (fv[w] | fs[w]) : 0u;
    uint32_t prev = __shfl_up_sync(LFPS_FULL, cur, 1);
    uint32_t next = __shfl_down_sync(LFPS_FULL, cur, 1);
    if (lane == 0) prev = (w > 0 && w - 1 < W) ? (c0v[w - 1] | c0s[w - 1]) : 0u;
    if (lane == 31) next = (w + 1 < W) ? (c0v[w + 1] | c0s[w + 1]) : 0u;
    uint32_t dil = 0;
    for (int k = 0; k < c.n_off; ++k) dil |= shifted(prev, cur, next, c.off[k]);
    const uint32_t valid = !in ? 0u : (w == W - 1 ? last_valid : LFPS_FULL);
    const uint32_t c1 = f & dil & valid;
    uint32_t tail = 0;
    const int j0 = w * 32;
    if (in && j0 + 32 > tail_lo) tail = (LFPS_FULL << max(0, tail_lo - j0)) & valid;
    const uint32_t pr = c1 | tail;
    if (in) pwords[w] = pr;
    n0 += __popc(cur);
    n1 += __popc(c1);
    nd += __popc(cur & ~c1);
    int bc = __popc(pr);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) bc += __shfl_xor_sync(LFPS_FULL, bc, o);
    if (lane == 0) blk[bk] = bc;
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    n0 += __shfl_xor_sync(LFPS_FULL, n0, o);
    n1 += __shfl_xor_sync(LFPS_FULL, n1, o);
    nd += __shfl_xor_sync(LFPS_FULL, nd, o);
  }
  if (lane == 0) { red[0][warp] = n0; red[1][warp] = n1; red[2][warp] = nd; }
  __syncthreads();
  if (warp == 0) {
    // exclusive scan of the block counts (nblk <= 192)
    int carry = 0;
    for (int base = 0; base < nblk; base += 32) {
      const int i = base + lane;
      const int v = i < nblk ? blk[i] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(LFPS_FULL, x, o);
        if (lane >= o) x += y;
      }
      if (i < nblk) blk[i] = carry + x - v;
      carry += __shfl_sync(LFPS_FULL, x, 31);
    }
    if (lane == 0) {
      int t0 = 0, t1 = 0, t3 = 0;
      for (int k = 0; k < kWarps; ++k) { t0 += red[0][k]; t1 += red[1][k]; t3 += red[2][k]; }
      cnt[CNT_C0] = t0;
      cnt[CNT_C1] = t1;
      cnt[CNT_PROBE] = carry;
      cnt[CNT_DROP] = t3;
    }
  }
  __syncthreads();
  // phase B: emit absolute indices in ascending order
  int* out = c.probe_idx + (size_t)s * c.list_cap;
  for (int bk = warp; bk < nblk; bk += kWarps) {
    const int w = bk * 32 + lane;
    uint32_t pr = w < W ? pwords[w] : 0u;
    const int pc = __popc(pr);
    int x = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(LFPS_FULL, x, o);
      if (lane >= o) x += y;
    }
    int pos = blk[bk] + x - pc;
    while (pr) {
      const int bit = __ffs(pr) - 1;
      out[pos++] = S + w * 32 + bit;
      pr &= pr - 1;
    }
  }
}

}  // namespace

cudaError_t launch_probe(const Ctx& c, cudaStream_t st) {
  const size_t smem = (size_t)c.words * 4;
  static int set = 0;
  if (!set) {
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    set = 1;
  }
  probe_kernel<<<c.NS, kThreads, smem, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
