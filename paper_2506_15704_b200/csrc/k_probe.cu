// k_probe.cu -- candidate construction (rest of K2): C0, C1, probe.
//
// Per session (one CTA):
//   C0 = {i : ver_p[i] > tau_v/scale} u {i : sla_p(i) > tau_s/scale}
//        (select_initial, candidates.py:45-58) -- rebuilt exactly from the
//        slots captured by k_tables.cu (or its fallback bitmap) into a
//        shared-memory bitmap;
//   C1 = F & dilate(C0, offsets) where dilate sets bit j when j - delta is in
//        C0, and F(j) = ver_p[j] > mean_v/scale or sla_p(j) > mean_s/scale is
//        read from the tables only at dilated positions (expand,
//        candidates.py:61-82, including delta = 0 being filtered);
//   probe = C1 | trailing local window (finalize_probe_set,
//        candidates.py:85-100), emitted as a sorted absolute index list.
// All comparisons are exact fp64 (on the bit patterns: phys values are +0 or
// positive, thresholds >= 0 or NaN).
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

__device__ __forceinline__ long long thr_bits(double t) {
  // values compared are +0 or positive: NaN never passes, -inf always passes
  if (isnan(t)) return 0x7fffffffffffffffll;
  if (t < 0.0) return -1ll;
  return __double_as_longlong(t);
}

__global__ void __launch_bounds__(kThreads) lfps_probe_kernel(Ctx c) {
  extern __shared__ uint32_t smem[];
  __shared__ int blk[512];
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
  uint32_t* c0w = smem;            // [W] C0 bitmap
  uint32_t* pwords = smem + W;     // [W] probe bitmap
  const double* itv = c.tb.itemf + (size_t)(2 * s) * 4;
  const double* its = c.tb.itemf + (size_t)(2 * s + 1) * 4;

  // ---- C0 -----------------------------------------------------------------
  if (c.exhaustive) {
    for (int w = tid; w < W; w += kThreads)
      c0w[w] = (w == W - 1 && (m & 31)) ? ((1u << (m & 31)) - 1u) : LFPS_FULL;
  } else {
    for (int w = tid; w < W; w += kThreads) {
      uint32_t v = 0;
      for (int t = 0; t < 2; ++t) {
        const int item = 2 * s + t;
        if (c.tb.fb[item]) v |= __ldcg(c.bits + (size_t)item * c.words + w);
      }
      c0w[w] = v;
    }
    __syncthreads();
    for (int t = 0; t < 2; ++t) {
      const int item = 2 * s + t;
      const double* itf = c.tb.itemf + (size_t)item * 4;
      if (c.tb.fb[item] || itf[2] != 0.0) continue;
      const long long tb = thr_bits(itf[0]);
      const int nc = min(c.tb.ncap[item], c.tb.cap);
      const int* ci = c.tb.cidx + (size_t)item * c.tb.cap;
      const double* cv = c.tb.cval + (size_t)item * c.tb.cap;
      for (int j = tid; j < nc; j += kThreads) {
        if (__double_as_longlong(__ldcg(cv + j)) > tb) {
          const int i = __ldcg(ci + j);
          atomicOr(&c0w[i >> 5], 1u << (i & 31));
        }
      }
    }
  }
  __syncthreads();

  // ---- C1 = F & dilate(C0); probe = C1 | tail ------------------------------------
  const long long tfv = thr_bits(itv[1]);
  const long long tfs = thr_bits(its[1]);
  const long long* ver = reinterpret_cast<const long long*>(c.ver + (size_t)s * c.m_cap);
  const long long* ring = reinterpret_cast<const long long*>(c.sla + (size_t)s * c.ring_cap);
  const int base = c.sla_base[s];
  const int C = c.ring_cap;
  const int tail_lo = max(0, m - c.L);
  const uint32_t last_valid = (m & 31) ? ((1u << (m & 31)) - 1u) : LFPS_FULL;
  int n0 = 0, n1 = 0, nd = 0;
  for (int bk = warp; bk < nblk; bk += kWarps) {
    const int w = bk * 32 + lane;
    const bool in = w < W;
    const uint32_t cur = in ? c0w[w] : 0u;
    const uint32_t prev = (in && w > 0) ? c0w[w - 1] : 0u;
    const uint32_t next = (in && w + 1 < W) ? c0w[w + 1] : 0u;
    uint32_t dil = 0;
    for (int k = 0; k < c.n_off; ++k) dil |= shifted(prev, cur, next, c.off[k]);
    const uint32_t valid = !in ? 0u : (w == W - 1 ? last_valid : LFPS_FULL);
    uint32_t cand = dil & valid;
    uint32_t c1 = 0;
    if (c.exhaustive) {
      c1 = cand;
    } else {
      // F at the dilated positions, four positions (eight loads) in flight
      while (cand) {
        int pos[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          pos[q] = cand ? __ffs(cand) - 1 : -1;
          cand &= cand - 1;
        }
        long long xv[4], xs[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xv[q] = xs[q] = -1ll;
          if (pos[q] >= 0) {
            const int i = w * 32 + pos[q];
            int p = base + i;
            if (p >= C) p -= C;
            xv[q] = __ldcg(ver + i);
            xs[q] = __ldcg(ring + p);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (pos[q] >= 0 && (xv[q] > tfv || xs[q] > tfs)) c1 |= 1u << pos[q];
      }
    }
    uint32_t tail = 0;
    const int j0 = w * 32;
    if (in && j0 + 32 > tail_lo) tail = (LFPS_FULL << max(0, tail_lo - j0)) & valid;
    const uint32_t pr = c1 | tail;
    if (in) pwords[w] = pr;
    if (in && (c.flags & LFPS_FLAG_EXPORT_SETS)) {
      c.bits[(size_t)(2 * s) * c.words + w] = cur;      // C0
      c.bits[(size_t)(2 * s + 1) * c.words + w] = c1;   // C1
    }
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
    int carry = 0;
    for (int base2 = 0; base2 < nblk; base2 += 32) {
      const int i = base2 + lane;
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

cudaError_t launch_probe(const Ctx& c, int m_max, cudaStream_t st) {
  const size_t smem = 2 * (size_t)((m_max + 31) / 32) * 4;
  static int set = 0;
  if (!set) {
    cudaFuncSetAttribute(lfps_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    set = 1;
  }
  lfps_probe_kernel<<<c.NS, kThreads, smem, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
