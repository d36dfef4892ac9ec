// tables.cuh -- the tracker-table statistics behind the thresholds and C0:
// canonical block moments, the pairwise merge tree and the hot-block scan
// (k_select.cu, k_update.cu).  See k_select.cu for the algorithm.
#pragma once

#include "common.cuh"
#include "canon.cuh"

namespace lfps {
namespace tbl {

constexpr int kLeaves = 512;                  // segments per window: m <= 511 * 512

struct Mom {
  double n, mu, m2, m3, m4;
};

// exact pairwise update (devmath.merge_moments), fixed op order
__device__ __forceinline__ Mom merge(const Mom& a, const Mom& b) {
  if (b.n == 0.0) return a;
  if (a.n == 0.0) return b;
  Mom r;
  r.n = cadd(a.n, b.n);
  const double delta = csub(b.mu, a.mu);
  const double dn = cdiv_count(delta, r.n);
  const double dn2 = cmul(dn, dn);
  const double t = cmul(cmul(cmul(delta, dn), a.n), b.n);
  r.mu = cadd(a.mu, cmul(b.n, dn));
  r.m2 = cadd(cadd(a.m2, b.m2), t);
  r.m3 = cadd(cadd(cadd(a.m3, b.m3), cmul(cmul(t, dn), csub(a.n, b.n))),
              cmul(cmul(3.0, dn), csub(cmul(a.n, b.m2), cmul(b.n, a.m2))));
  const double nn = cadd(csub(cmul(a.n, a.n), cmul(a.n, b.n)), cmul(b.n, b.n));
  r.m4 = cadd(cadd(cadd(cadd(a.m4, b.m4), cmul(cmul(t, dn2), nn)),
                   cmul(cmul(6.0, dn2), cadd(cmul(cmul(a.n, a.n), b.m2), cmul(cmul(b.n, b.n), a.m2)))),
              cmul(cmul(4.0, dn), csub(cmul(a.n, b.m3), cmul(b.n, a.m3))));
  return r;
}

__device__ __forceinline__ Mom shfl_mom(const Mom& a, int mask) {
  Mom r;
  r.n = __shfl_xor_sync(LFPS_FULL, a.n, mask);
  r.mu = __shfl_xor_sync(LFPS_FULL, a.mu, mask);
  r.m2 = __shfl_xor_sync(LFPS_FULL, a.m2, mask);
  r.m3 = __shfl_xor_sync(LFPS_FULL, a.m3, mask);
  r.m4 = __shfl_xor_sync(LFPS_FULL, a.m4, mask);
  return r;
}

// an item's window [lo, lo + m) of table slots and its blocks
struct Window {
  int lo, m, first, nseg;
};

__device__ __forceinline__ Window make_window(int lo, int m) {
  Window w;
  w.lo = lo;
  w.m = m;
  w.first = lo / kBlk;
  w.nseg = (lo + m - 1) / kBlk - w.first + 1;
  return w;
}

// segment of block blk: slots [a, a + vc)
__device__ __forceinline__ void segment(const Window& w, int blk, int& a, int& vc) {
  a = max(blk * kBlk, w.lo);
  vc = min(blk * kBlk + kBlk, w.lo + w.m) - a;
}

// element j of the segment -> lane j % 32, position j / 32 (0 beyond vc)
__device__ __forceinline__ void load_seg(const double* row, int a, int vc, int lane, double* v) {
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const int j = e * 32 + lane;
    v[e] = j < vc ? __ldg(row + a + j) : 0.0;   // tables are read-only here: L1 path
  }
}

// segment mean and centred power sums (devmath.chunk_moments)
template <bool FULL>
__device__ __forceinline__ void seg_moments(const double* v, int vc, int lane, double& mu,
                                            double& m2, double& m3, double& m4) {
  double q[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) q[g] = cadd(cadd(v[4 * g], v[4 * g + 1]), cadd(v[4 * g + 2], v[4 * g + 3]));
  const double sum = warp_fold(cadd(cadd(q[0], q[1]), cadd(q[2], q[3])));
  mu = FULL ? cmul(sum, 1.0 / 512.0) : cdiv_count(sum, (double)vc);
  double p2[4], p3[4], p4[4];
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    double t2[4], t3[4], t4[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int e = 4 * g + t;
      const double d = (FULL || e * 32 + lane < vc) ? csub(v[e], mu) : 0.0;
      const double d2 = cmul(d, d);
      t2[t] = d2;
      t3[t] = cmul(d2, d);
      t4[t] = cmul(d2, d2);
    }
    p2[g] = cadd(cadd(t2[0], t2[1]), cadd(t2[2], t2[3]));
    p3[g] = cadd(cadd(t3[0], t3[1]), cadd(t3[2], t3[3]));
    p4[g] = cadd(cadd(t4[0], t4[1]), cadd(t4[2], t4[3]));
  }
  m2 = warp_fold(cadd(cadd(p2[0], p2[1]), cadd(p2[2], p2[3])));
  m3 = warp_fold(cadd(cadd(p3[0], p3[1]), cadd(p3[2], p3[3])));
  m4 = warp_fold(cadd(cadd(p4[0], p4[1]), cadd(p4[2], p4[3])));
}

// canonical merge of one quarter of the window's segments: the pairwise tree
// over 512 leaves (leaf i = segment i) is four 128-leaf subtrees merged
// ((q0, q1), (q2, q3)); warp quarter qd owns leaves [128 qd, 128 qd + 128),
// lane l the four leaves [128 qd + 4 l, + 4)
__device__ __forceinline__ Mom leaf(const double* bs, const Window& w, int i) {
  Mom r = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (i < w.nseg) {
    int a, vc;
    segment(w, w.first + i, a, vc);
    r.n = (double)vc;
    const double2* p = reinterpret_cast<const double2*>(bs + 4 * (size_t)(w.first + i));
    const double2 x = __ldcg(p), y = __ldcg(p + 1);
    r.mu = x.x; r.m2 = x.y; r.m3 = y.x; r.m4 = y.y;
  }
  return r;
}

__device__ __forceinline__ Mom quarter_merge(const double* bs, Window w, int qd, int lane) {
  const int i0 = qd * 128 + lane * 4;
  Mom acc = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (i0 < w.nseg) {
    const Mom a = merge(leaf(bs, w, i0), leaf(bs, w, i0 + 1));
    const Mom b = merge(leaf(bs, w, i0 + 2), leaf(bs, w, i0 + 3));
    acc = merge(a, b);
  }
#pragma unroll
  for (int h = 1; h <= 16; h <<= 1) {
    const Mom o = shfl_mom(acc, h);
    acc = (lane & h) ? merge(o, acc) : merge(acc, o);
  }
  return acc;
}

// exclusive scan over the 256 threads of the block; total in *total
__device__ __forceinline__ long long thr_bits(double t) {
  // values compared are +0 or positive: NaN never passes, -inf always passes
  if (isnan(t)) return 0x7fffffffffffffffll;
  if (t < 0.0) return -1ll;
  return __double_as_longlong(t);
}

__device__ __forceinline__ long long warp_max64(long long x) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) x = max(x, (long long)__shfl_xor_sync(LFPS_FULL, x, o));
  return x;
}

struct StatsShared {
  int ntask, nhot, npair;
  int task[kLeaves];
  int hot[kLeaves];
  Mom part[4];
  double thr0;
  int deg;
};

// C0 words of one (session, table), written by lfps_stats_kernel for
// lfps_select_kernel (ws.hot): entry 0 = (count, 0), then (logical index of
// the word's first slot, 32 slot bits); at most 16 words per block
__device__ __forceinline__ int2* hot_list(const Ctx& c, int s, int t) {
  return c.hot + (size_t)(2 * s + t) * (16 * c.bw.nblk + 1);
}

// named barrier of one 128-thread table worker (ids 1.. ; 0 is __syncthreads)
__device__ __forceinline__ void worker_sync(int bar) {
  asm volatile("bar.sync %0, 128;" ::"r"(bar) : "memory");
}

// A + B + C of table t of session s by one 128-thread worker (tid4 in
// [0, 128), its 4 warps), for the window w at scale sc:
//   A  rebuild the blocks flagged by dirty_word(i) (i < dwords; all of the
//      window's blocks when `full`);
//   B  the canonical merge tree -> thr_next[(2 s + t) * 4 + {tau, mean, deg,
//      kappa}] (kappa == 0 is raised by the select kernel);
//   C  the table's C0 words -> hot_list(c, s, t), entry 0 = (words, blocks read).
// bar: the worker's named barrier (the worker's threads only).
template <typename DirtyWord>
__device__ void maintain_table(const Ctx& c, int s, int t, const Window& w, double sc, bool full,
                               DirtyWord dirty_word, StatsShared& sh, int tid4, int bar,
                               long long tclk0) {
  const int lane = tid4 & 31, warp = tid4 >> 5;
  const int nb = c.bw.nblk;
  const int dw = c.bw.dwords;
  const double* row = t ? sla_row(c, s) : ver_row(c, s);

  // ---- A: rebuild dirty blocks ------------------------------------------------------
  if (tid4 == 0) sh.ntask = 0;
  worker_sync(bar);
  if (tid4 < dw) {
    uint32_t bits = full ? LFPS_FULL : dirty_word(tid4);
    const int lo = w.first - tid4 * 32, hi = w.first + w.nseg - tid4 * 32;   // window blocks
    const uint32_t in_lo = lo <= 0 ? LFPS_FULL : (lo >= 32 ? 0u : (LFPS_FULL << lo));
    const uint32_t in_hi = hi >= 32 ? LFPS_FULL : (hi <= 0 ? 0u : (LFPS_FULL >> (32 - hi)));
    bits &= in_lo & in_hi;
    if (bits) {
      int pos = atomicAdd(&sh.ntask, __popc(bits));
      while (bits) {
        const int k = __ffs(bits) - 1;
        bits &= bits - 1;
        sh.task[pos++] = tid4 * 32 + k;
      }
    }
  }
  worker_sync(bar);
  for (int k = warp; k < sh.ntask; k += 4) {
    const int blk = sh.task[k];
    int a, vc;
    segment(w, blk, a, vc);
    double v[16];
    load_seg(row, a, vc, lane, v);
    double mu, m2, m3, m4;
    if (vc == kBlk) seg_moments<true>(v, vc, lane, mu, m2, m3, m4);
    else seg_moments<false>(v, vc, lane, mu, m2, m3, m4);
    long long mx = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e)
      if (e * 32 + lane < vc) mx = max(mx, __double_as_longlong(v[e]));
    mx = warp_max64(mx);
    if (lane == 0) {
      const size_t it = (size_t)(2 * s + t) * nb + blk;
      double2* p = reinterpret_cast<double2*>(c.bw.bsum + 4 * it);
      p[0] = make_double2(mu, m2);
      p[1] = make_double2(m3, m4);
      c.bw.bmax[it] = __longlong_as_double(mx);
    }
  }
  worker_sync(bar);
  if (t == 0) trace_at(c, s, 1, tclk0);

  // the window's block maxima (C's input, final after A) load during B
  long long bmx[kLeaves / 128];
  {
    const double* bm = c.bw.bmax + (size_t)(2 * s + t) * nb + w.first;
#pragma unroll
    for (int k = 0; k < kLeaves / 128; ++k) {
      const int i = tid4 + 128 * k;
      bmx[k] = i < w.nseg ? __double_as_longlong(__ldcg(bm + i)) : 0ll;
    }
  }
  // ---- B: thresholds (compute_thresholds), one quarter of the tree per warp ----------
  const Mom q = quarter_merge(c.bw.bsum + (size_t)(2 * s + t) * nb * 4, w, warp, lane);
  if (lane == 0) sh.part[warp] = q;
  worker_sync(bar);
  if (tid4 == 0) {
    const Mom tot = merge(merge(sh.part[0], sh.part[1]), merge(sh.part[2], sh.part[3]));
    const double mean = cmul(tot.mu, sc);
    const bool deg = cmul(cmul(tot.m2, sc), sc) < 1e-12;
    double tau = NAN, kappa = NAN;
    if (!deg) {
      kappa = cdiv(tot.m4, cmul(tot.m2, tot.m2));
      tau = cdiv(cmul(c.a, mean), kappa);
    }
    double* thr = c.thr_next + (size_t)(2 * s + t) * 4;
    thr[0] = tau; thr[1] = mean; thr[2] = deg ? 1.0 : 0.0; thr[3] = kappa;
    sh.deg = deg ? 1 : 0;
    sh.thr0 = deg ? NAN : cdiv(tau, sc);
    sh.nhot = 0;
    sh.npair = 0;
    if (t == 0 && (c.flags & LFPS_FLAG_TRACE)) c.trace[(size_t)s * 16 + 2] = now_clk() - tclk0;
  }
  worker_sync(bar);

  // ---- C: this table's part of C0 (select_initial): only blocks whose max is
  // above tau / scale can hold members (the dirty ones were just read by A) ----
  int2* hot = hot_list(c, s, t);
  if (!sh.deg) {
    const long long tb = thr_bits(sh.thr0);
#pragma unroll
    for (int k = 0; k < kLeaves / 128; ++k) {
      const int i = tid4 + 128 * k;
      if (i < w.nseg && bmx[k] > tb) sh.hot[atomicAdd(&sh.nhot, 1)] = w.first + i;
    }
    worker_sync(bar);
    for (int k = warp; k < sh.nhot; k += 4) {
      const int blk = sh.hot[k];
      int a, vc;
      segment(w, blk, a, vc);
      double v[16];
      load_seg(row, a, vc, lane, v);
      const int L0 = a - w.lo;                         // logical index of element 0
      uint32_t mine = 0;                               // lane e keeps ballot word e
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const uint32_t wd = __ballot_sync(LFPS_FULL, e * 32 + lane < vc &&
                                                         __double_as_longlong(v[e]) > tb);
        if (lane == e) mine = wd;
      }
      if (lane < 16 && mine) hot[1 + atomicAdd(&sh.npair, 1)] = make_int2(L0 + lane * 32, (int)mine);
    }
    worker_sync(bar);
  }
  if (tid4 == 0) {
    hot[0] = make_int2(sh.npair, sh.ntask + sh.nhot);
    if (t == 0 && (c.flags & LFPS_FLAG_TRACE)) c.trace[(size_t)s * 16 + 7] = now_clk() - tclk0;
  }
}

}  // namespace tbl
}  // namespace lfps
