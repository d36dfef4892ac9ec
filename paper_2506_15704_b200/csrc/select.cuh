// select.cuh -- C0 assembly and candidate construction (C + D) of one
// session, as a device function of a 256-thread CTA: the body of
// lfps_select_kernel (k_select.cu) and the front half of the fused
// select + finish kernel (k_finish.cu).  See k_select.cu for the algorithm.
#pragma once

#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"
#include "tables.cuh"

namespace lfps {
namespace sel {

using namespace tbl;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef LFPS_SEL_DEPTH
#define LFPS_SEL_DEPTH 4
#endif
constexpr int kSelDepth = LFPS_SEL_DEPTH;   // F reads in flight per thread

// exclusive scan over the 256 threads of the block; total in *total
__device__ __forceinline__ int block_scan(int v, int* warp_sums, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(LFPS_FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  int before = 0, all = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    const int ws = warp_sums[k];
    before += k < warp ? ws : 0;
    all += ws;
  }
  __syncthreads();
  *total = all;
  return before + x - v;
}

// bits of C0 at positions j - delta for j in word w (|delta| <= 31)
__device__ __forceinline__ uint32_t shifted(uint32_t prev, uint32_t cur, uint32_t next, int delta) {
  if (delta == 0) return cur;
  if (delta > 0) return (cur << delta) | (prev >> (32 - delta));
  const int k = -delta;
  return (cur >> k) | (next << (32 - k));
}

// Top-k budget k = max(1, round_half_even(frac * n)) (engine.py:167)
__device__ __forceinline__ int unit_budget(const Ctx& c, int n) {
  const int k = (int)rint(c.frac * (double)n);
  return k < 1 ? 1 : k;
}

struct SelectShared {
  double thr0[2], thrf[2];
  int deg[2];
  int wsum[kWarps];
  int red[3][kWarps];
};

// dynamic shared memory of select_session for W = ceil(m / 32) C0 words:
// C0 bitmap [W], active-word list [W] u16, active words [ceil(W / 32)],
// then the flattening buffers (u16 [256 * 32], int [256], u32 [256])
__host__ __device__ constexpr size_t select_bitmap_bytes(int W) {
  return ((size_t)W * 4 + (size_t)(W + 1) / 2 * 4 + (size_t)(W + 31) / 32 * 4 + 15) / 16 * 16;
}
__host__ __device__ constexpr size_t select_smem(int m_max) {
  return select_bitmap_bytes((m_max + 31) / 32) + kThreads * 32 * 2 + kThreads * 4 * 2;
}

// C + D of session s from the thresholds and C0 words of lfps_stats_kernel;
// smem: select_smem(m_max) bytes of dynamic shared memory.
__device__ __forceinline__ void select_session(const Ctx& c, int s, uint32_t* smem,
                                               SelectShared& sh) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* cnt = c.counts + (size_t)s * CNT_N;
  const int b = s / c.Hq;
  // independent prologue loads, issued together (one round trip, not four)
  const int byp = c.prefetch ? 0 : c.bypass[s];   // run ahead of the gate: every session
  const int n = c.n_ctx[b];
  const int base = c.sla_base[s];
  double tau = 0.0, mean = 0.0, degv = 0.0, kap = 0.0, sc = 1.0;
  if (tid < 2 && !c.exhaustive) {
    const double* thr = c.thr_next + (size_t)(2 * s + tid) * 4;
    tau = thr[0]; mean = thr[1]; degv = thr[2]; kap = thr[3];
    sc = c.scale[s];
  }
  // the tables' C0 words from lfps_stats_kernel: the counts and the first
  // 256 words of each list in the same round trip
  int2 hp[2] = {make_int2(0, 0), make_int2(0, 0)};
  int hn[2] = {0, 0}, blocks = 0;
  if (!c.exhaustive) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int2* hl = hot_list(c, s, t);
      const int2 h0 = hl[0];
      hn[t] = h0.x;
      blocks += h0.y;
      if (tid < 16 * c.bw.nblk) hp[t] = hl[1 + tid];
    }
  }
  if (tid == 0 && !c.exhaustive) atomicMax(c.bw.valid + s, 1);   // summaries current (2: + thresholds)
  if (byp) {
    if (tid < CNT_N) cnt[tid] = tid == CNT_BLOCKS ? blocks : 0;
    return;
  }
  const int S = c.S;
  const int m = n - S;
  const int W = (m + 31) / 32;
  uint32_t* c0w = smem;                      // [W] C0 bitmap (logical index)
  uint16_t* alist = reinterpret_cast<uint16_t*>(smem + W);   // [W] active word list
  uint32_t* act = smem + W + (W + 1) / 2;    // [AW] active words (C0 word +- 1, tail)
  const int AW = (W + 31) / 32;
  // candidate flattening buffers behind the bitmaps (16-B aligned)
  uint8_t* fb = reinterpret_cast<uint8_t*>(smem) + select_bitmap_bytes(W);
  uint16_t* fbuf = reinterpret_cast<uint16_t*>(fb);          // [kThreads * 32]
  int* fword = reinterpret_cast<int*>(fb + kThreads * 32 * 2);   // [kThreads]
  uint32_t* fc1 = reinterpret_cast<uint32_t*>(fword + kThreads); // [kThreads]
  const double* ver = ver_row(c, s);
  const double* sla = sla_row(c, s) + base;   // logical view
  const Window wv = make_window(0, m);
  const Window wsl = make_window(base, m);
  const long long tclk0 = now_clk();

  for (int w = tid; w < W; w += kThreads)
    c0w[w] = !c.exhaustive ? 0u : ((w == W - 1 && (m & 31)) ? ((1u << (m & 31)) - 1u) : LFPS_FULL);
  for (int w = tid; w < AW; w += kThreads)
    act[w] = !c.exhaustive ? 0u : ((w == AW - 1 && (W & 31)) ? ((1u << (W & 31)) - 1u) : LFPS_FULL);
  if (tid < 2) {
    const int t = tid;
    double* thr = c.thr + (size_t)(2 * s + t) * 4;
    if (c.exhaustive) {
      sh.thr0[t] = -INFINITY; sh.thrf[t] = -INFINITY; sh.deg[t] = 0;
      thr[0] = -INFINITY; thr[1] = -INFINITY; thr[2] = 0.0; thr[3] = NAN;
    } else {
      sh.deg[t] = degv != 0.0;
      sh.thr0[t] = sh.deg[t] ? NAN : cdiv(tau, sc);
      sh.thrf[t] = cdiv(mean, sc);
      thr[0] = tau; thr[1] = mean; thr[2] = degv; thr[3] = kap;   // export
      if (!sh.deg[t] && kap == 0.0 && !c.prefetch) set_err(c, s, LFPS_ERR_KAPPA_ZERO);
    }
  }
  __syncthreads();
  if (tid == 0 && !c.exhaustive) {       // tail words are always active
    for (int w = max(0, m - c.L) >> 5; w < W; ++w) act[w >> 5] |= 1u << (w & 31);
  }
  // ---- C: C0 = union of the tables' words (select_initial) ------------------------
  if (!c.exhaustive) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int2* hl = hot_list(c, s, t);
      for (int i = tid; i < hn[t]; i += kThreads) {
        const int2 e = i == tid ? hp[t] : hl[1 + i];
        const uint32_t mine = (uint32_t)e.y;
        const int L = e.x;
        const int sft = L & 31, wi = L >> 5;
        atomicOr(&c0w[wi], mine << sft);
        const bool hi = sft && (mine >> (32 - sft));
        if (hi) atomicOr(&c0w[wi + 1], mine >> (32 - sft));
        // the words whose dilation can see these bits become active
        for (int x = max(0, wi - 1); x <= min(W - 1, wi + (hi ? 2 : 1)); ++x)
          atomicOr(&act[x >> 5], 1u << (x & 31));
      }
    }
    __syncthreads();
  }

  trace_at(c, s, 3, tclk0);
  // ---- D: C1 = F & dilate(C0); probe = C1 | tail, over the active words only ----
  {
    int na;
    const uint32_t aw = tid < AW ? act[tid] : 0u;      // AW <= 256
    int pos = block_scan(__popc(aw), sh.wsum, &na);
    for (uint32_t x = aw; x; x &= x - 1) alist[pos++] = (uint16_t)(tid * 32 + __ffs(x) - 1);
    if (c.flags & LFPS_FLAG_EXPORT_SETS) {
      for (int w = tid; w < W; w += kThreads) {
        c.bits[(size_t)(2 * s) * c.words + w] = c0w[w];   // C0
        c.bits[(size_t)(2 * s + 1) * c.words + w] = 0u;   // C1 (active words below)
      }
    }
    __syncthreads();
    const long long tfv = thr_bits(sh.thrf[0]);
    const long long tfs = thr_bits(sh.thrf[1]);
    const long long* verb = reinterpret_cast<const long long*>(ver);
    const long long* slab = reinterpret_cast<const long long*>(sla);
    const int tail_lo = max(0, m - c.L);
    const uint32_t last_valid = (m & 31) ? ((1u << (m & 31)) - 1u) : LFPS_FULL;
    int* out = c.probe_idx + (size_t)s * c.list_cap;
    int n0 = 0, n1 = 0, nd = 0, written = 0;
    for (int r = 0; r < na; r += kThreads) {
      const int j = r + tid;
      const int w = j < na ? alist[j] : -1;
      uint32_t cur = 0u, cand = 0u, valid = LFPS_FULL;
      if (w >= 0) {
        cur = c0w[w];
        const uint32_t prev = w > 0 ? c0w[w - 1] : 0u;
        const uint32_t next = w + 1 < W ? c0w[w + 1] : 0u;
        uint32_t dil = 0;
        for (int k = 0; k < c.n_off; ++k) dil |= shifted(prev, cur, next, c.off[k]);
        valid = w == W - 1 ? last_valid : LFPS_FULL;
        cand = dil & valid;
      }
      uint32_t c1 = cand;
      if (!c.exhaustive) {
        // F at the dilated positions.  The round's candidates are flattened
        // into one list and read by all 256 threads, 4 deep: a band of dense
        // words (32 candidates each, all in one warp) costs no more round
        // trips than scattered sparse words.
        int K;
        int off = block_scan(__popc(cand), sh.wsum, &K);
        for (uint32_t x = cand; x; x &= x - 1) fbuf[off++] = (uint16_t)((tid << 5) | (__ffs(x) - 1));
        fword[tid] = w;
        fc1[tid] = 0u;
        __syncthreads();
        for (int g0 = tid; g0 < K; g0 += kSelDepth * kThreads) {
          int e[kSelDepth];
          long long xv[kSelDepth], xs[kSelDepth];
#pragma unroll
          for (int q = 0; q < kSelDepth; ++q) e[q] = g0 + kThreads * q < K ? fbuf[g0 + kThreads * q] : -1;
#pragma unroll
          for (int q = 0; q < kSelDepth; ++q) {
            xv[q] = xs[q] = -1ll;
            if (e[q] >= 0) {
              const int i = fword[e[q] >> 5] * 32 + (e[q] & 31);
              xv[q] = __ldg(verb + i);
              xs[q] = __ldg(slab + i);
            }
          }
#pragma unroll
          for (int q = 0; q < kSelDepth; ++q)
            if (e[q] >= 0 && (xv[q] > tfv || xs[q] > tfs))
              atomicOr(&fc1[e[q] >> 5], 1u << (e[q] & 31));
        }
        __syncthreads();
        if (r == 0) trace_at(c, s, 6, tclk0);         // first round's F reads done
        c1 = fc1[tid];
      }
      uint32_t pr = 0u;
      if (w >= 0) {
        uint32_t tail = 0;
        const int j0 = w * 32;
        if (j0 + 32 > tail_lo) tail = (LFPS_FULL << max(0, tail_lo - j0)) & valid;
        pr = c1 | tail;
        if (c.flags & LFPS_FLAG_EXPORT_SETS) c.bits[(size_t)(2 * s + 1) * c.words + w] = c1;
        n0 += __popc(cur);
        n1 += __popc(c1);
        nd += __popc(cur & ~c1);
      }
      int tot;
      int at = written + block_scan(__popc(pr), sh.wsum, &tot);
      for (; pr; pr &= pr - 1) out[at++] = S + w * 32 + __ffs(pr) - 1;
      written += tot;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      n0 += __shfl_xor_sync(LFPS_FULL, n0, o);
      n1 += __shfl_xor_sync(LFPS_FULL, n1, o);
      nd += __shfl_xor_sync(LFPS_FULL, nd, o);
    }
    if (lane == 0) { sh.red[0][warp] = n0; sh.red[1][warp] = n1; sh.red[2][warp] = nd; }
    __syncthreads();
    if (tid == 0) {
      int t0 = 0, t1 = 0, t3 = 0;
      for (int k = 0; k < kWarps; ++k) { t0 += sh.red[0][k]; t1 += sh.red[1][k]; t3 += sh.red[2][k]; }
      cnt[CNT_C0] = t0;
      cnt[CNT_C1] = t1;
      cnt[CNT_PROBE] = written;
      cnt[CNT_DROP] = t3;
      cnt[CNT_BLOCKS] = blocks;
      if (c.flags & LFPS_FLAG_TRACE) {
        c.trace[(size_t)s * 16 + 4] = now_clk() - tclk0;
        c.trace[(size_t)s * 16 + 12] = now_ns();
      }
    }
  }
}


}  // namespace sel
}  // namespace lfps
