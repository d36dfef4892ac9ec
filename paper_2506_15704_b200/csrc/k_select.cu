// k_select.cu -- thresholds and candidate construction (K1 + K2) from
// PERSISTENT block summaries, as two kernels:
//
//   lfps_stats_kernel   one 128-thread CTA per (session, table): A + B
//   lfps_select_kernel  one 256-thread CTA per session: C + D
//
// Restates compute_thresholds (tables.py:295-317, _phys_moments :127-140),
// select_initial (candidates.py:45-58), expand (:61-82) and
// finalize_probe_set (:85-100).
//
// Each table is cut into 512-slot blocks of table slots (vertical: slot =
// logical index; slash: slot = sla_base + logical index, a window that only
// grows at its ends).  Every block carries a summary of its part of the
// window: the canonical segment moments (mean, M2, M3, M4) and the maximum
// phys value.  A decode step changes a table only at its C2 slots and at the
// one slot it grows by (k_update.cu marks those blocks dirty), and the lazy
// scale leaves phys values alone, so the summaries of all other blocks stay
// exact.  Per step
//
//   A  rebuilds the dirty blocks (every block when the session's summaries
//      are not valid: first step, after a renormalisation);
//   B  merges the window's segment moments in the canonical pairwise tree
//      (devmath.table_moments) -> tau, mean, degenerate, kappa in thr[];
//      exactly the same arithmetic as rebuilding every block;
//   C  C0 = {slots with phys > tau / scale}: only "hot" blocks (max above
//      the threshold) can hold members, and only those are read;
//   D  C1 = F & dilate(C0, offsets), F read at dilated slots only;
//      probe = C1 | local tail, compacted into a sorted absolute index list.
//
// A + B are fp64 latency chains per table: running them per (session, table)
// in 128-thread CTAs (8 per SM) doubles the sessions in flight over one
// 256-thread CTA per session doing both tables.
//
// All comparisons are exact fp64 (on bit patterns: phys values are +0 or
// positive).  Table bytes read per step: dirty + hot blocks, not 2 m.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
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

#ifndef LFPS_STATS_CTAS
#define LFPS_STATS_CTAS 8
#endif
#ifndef LFPS_SELECT_CTAS
#define LFPS_SELECT_CTAS 5
#endif
constexpr int kStatsThreads = 128;
constexpr int kStatsWarps = kStatsThreads / 32;

// A + B + C of one (session, table): rebuild the dirty blocks, merge the
// window's segment moments into thr_next[(2 s + t) * 4 + {tau, mean, deg,
// kappa}], and list the table's C0 words.
__global__ void __launch_bounds__(kStatsThreads, LFPS_STATS_CTAS) lfps_stats_kernel(Ctx c) {
  __shared__ StatsShared sh;
  const int s = c.s_off + (blockIdx.x >> 1), t = blockIdx.x & 1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (c.exhaustive) return;
  const int b = s / c.Hq;
  const int dw = c.bw.dwords;
  // independent prologue loads, issued together (one round trip, not four).
  // The stats kernel runs concurrently with the gate, so it works for every
  // session, gated or not: a gated session's thresholds are simply not used
  // (and not exported) by the select kernel.
  const int n = c.n_ctx[b];
  const int base = t ? c.sla_base[s] : 0;
  const bool valid = c.bw.valid[s] != 0;
  uint32_t* dp = c.bw.dirty + (size_t)(2 * s + t) * dw + tid;
  const uint32_t dbits = tid < dw ? *dp : 0u;
  const int m = n - c.S;
  const Window w = make_window(base, m);
  const int nb = c.bw.nblk;
  const double* row = t ? sla_row(c, s) : ver_row(c, s);
  const long long tclk0 = now_clk();
  if ((c.flags & LFPS_FLAG_TRACE) && tid == 0 && t == 0) c.trace[(size_t)s * 16 + 15] = now_ns();

  // ---- A: rebuild dirty blocks ------------------------------------------------------
  if (tid == 0) sh.ntask = 0;
  __syncthreads();
  if (tid < dw) {
    uint32_t bits = valid ? dbits : LFPS_FULL;
    if (bits) *dp = 0u;                             // also clears stale marks of a rebuild
    const int lo = w.first - tid * 32, hi = w.first + w.nseg - tid * 32;   // window blocks
    const uint32_t in_lo = lo <= 0 ? LFPS_FULL : (lo >= 32 ? 0u : (LFPS_FULL << lo));
    const uint32_t in_hi = hi >= 32 ? LFPS_FULL : (hi <= 0 ? 0u : (LFPS_FULL >> (32 - hi)));
    bits &= in_lo & in_hi;
    if (bits) {
      int pos = atomicAdd(&sh.ntask, __popc(bits));
      while (bits) {
        const int k = __ffs(bits) - 1;
        bits &= bits - 1;
        sh.task[pos++] = tid * 32 + k;
      }
    }
  }
  __syncthreads();
  for (int k = warp; k < sh.ntask; k += kStatsWarps) {
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
  __syncthreads();
  if (t == 0) trace_at(c, s, 1, tclk0);

  // ---- B: thresholds (compute_thresholds), one quarter of the tree per warp ----------
  const Mom q = quarter_merge(c.bw.bsum + (size_t)(2 * s + t) * nb * 4, w, warp, lane);
  if (lane == 0) sh.part[warp] = q;
  __syncthreads();
  if (tid == 0) {
    const Mom tot = merge(merge(sh.part[0], sh.part[1]), merge(sh.part[2], sh.part[3]));
    const double sc = c.scale[s];
    const double mean = cmul(tot.mu, sc);
    const bool deg = cmul(cmul(tot.m2, sc), sc) < 1e-12;
    double tau = NAN, kappa = NAN;
    if (!deg) {
      kappa = cdiv(tot.m4, cmul(tot.m2, tot.m2));   // kappa == 0 is raised by select
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
  __syncthreads();

  // ---- C: this table's part of C0 (select_initial): only blocks whose max is
  // above tau / scale can hold members (the dirty ones were just read by A) ----
  int2* hot = hot_list(c, s, t);
  if (!sh.deg) {
    const long long tb = thr_bits(sh.thr0);
    const double* bm = c.bw.bmax + (size_t)(2 * s + t) * nb;
    for (int i = tid; i < w.nseg; i += kStatsThreads)
      if (__double_as_longlong(__ldcg(bm + w.first + i)) > tb) sh.hot[atomicAdd(&sh.nhot, 1)] = w.first + i;
    __syncthreads();
    for (int k = warp; k < sh.nhot; k += kStatsWarps) {
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
    __syncthreads();
  }
  if (tid == 0) {
    hot[0] = make_int2(sh.npair, sh.ntask + sh.nhot);
    if (t == 0 && (c.flags & LFPS_FLAG_TRACE)) c.trace[(size_t)s * 16 + 7] = now_clk() - tclk0;
  }
}

struct SelectShared {
  uint16_t fbuf[kThreads * 32];  // the round's candidate slots: thread << 5 | bit
  int fword[kThreads];           // C0 word of each thread
  uint32_t fc1[kThreads];        // C1 bits of each thread's word
  double thr0[2], thrf[2];
  int deg[2];
  int wsum[kWarps];
  int red[3][kWarps];
};

// C + D of one session from the thresholds of lfps_stats_kernel.
__global__ void __launch_bounds__(kThreads, LFPS_SELECT_CTAS) lfps_select_kernel(Ctx c) {
  extern __shared__ uint32_t smem[];
  __shared__ SelectShared sh;
  const int s = c.s_off + blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* cnt = c.counts + (size_t)s * CNT_N;
  const int b = s / c.Hq;
  // independent prologue loads, issued together (one round trip, not four)
  const int byp = c.bypass[s];
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
  if (tid == 0 && !c.exhaustive) c.bw.valid[s] = 1;   // both tables' summaries are current
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
      if (!sh.deg[t] && kap == 0.0) set_err(c, s, LFPS_ERR_KAPPA_ZERO);
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
        for (uint32_t x = cand; x; x &= x - 1) sh.fbuf[off++] = (uint16_t)((tid << 5) | (__ffs(x) - 1));
        sh.fword[tid] = w;
        sh.fc1[tid] = 0u;
        __syncthreads();
        for (int g0 = tid; g0 < K; g0 += 4 * kThreads) {
          int e[4];
          long long xv[4], xs[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) e[q] = g0 + kThreads * q < K ? sh.fbuf[g0 + kThreads * q] : -1;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            xv[q] = xs[q] = -1ll;
            if (e[q] >= 0) {
              const int i = sh.fword[e[q] >> 5] * 32 + (e[q] & 31);
              xv[q] = __ldg(verb + i);
              xs[q] = __ldg(slab + i);
            }
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            if (e[q] >= 0 && (xv[q] > tfv || xs[q] > tfs))
              atomicOr(&sh.fc1[e[q] >> 5], 1u << (e[q] & 31));
        }
        __syncthreads();
        if (r == 0) trace_at(c, s, 6, tclk0);         // first round's F reads done
        c1 = sh.fc1[tid];
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

}  // namespace

cudaError_t launch_stats(const Ctx& c, cudaStream_t st) {
  lfps_stats_kernel<<<2 * c.s_cnt, kStatsThreads, 0, st>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_select(const Ctx& c, int m_max, cudaStream_t st) {
  const int W = (m_max + 31) / 32;
  const size_t smem = ((size_t)W + (W + 1) / 2 + (W + 31) / 32) * 4;
  static bool set = false;
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(lfps_select_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(lfps_select_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    set = true;
  }
  lfps_select_kernel<<<c.s_cnt, kThreads, smem, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
