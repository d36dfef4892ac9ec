// k_stages.cu -- the reference's per-head stage functions on the device, at
// the reference's precision (fp64 K/V, tables, logits and softmax).
//
// The batched decode step (k_gate / k_select / k_finish / k_update) fuses the
// stages of Algorithm 1 across B x Hq sessions with bf16 K/V and fp32 probe
// scores.  The reference package also exposes every stage on its own, on one
// head's float64 state (pkg/src/lfps/__init__.py:13-58): thresholds, the
// three candidate stages, restricted Top-k, attention output, the table
// update and growth, the Eq. 4 seeding, the head priors and the gate.  These
// kernels are those stages, one launch each, for one head (a reference
// HeadSession): generic d, fp64 everywhere, and the same canonical orders
// as the batched kernels where the two share a quantity (table moments:
// tables.cuh; fp64 dots: lanes strided over d, fold 16..1; devmath.gdot).
// One CTA per call unless stated: they serve the per-head API, not the
// batched hot path.
#include "common.cuh"
#include "canon.cuh"
#include "tables.cuh"

namespace lfps {
namespace {

constexpr int kT = 256;
constexpr int kW = kT / 32;

// canonical fp64 dot of one row with q by one warp (devmath.gdot)
__device__ __forceinline__ double gdot_warp(const double* row, const double* q, int d, int lane) {
  double acc = 0.0;
  for (int j = lane; j < d; j += 32) acc = cadd(acc, cmul(row[j], q[j]));
  return warp_fold(acc);
}

// ordered stream compaction of flagged positions [0, n) by one CTA: emit(pos,
// i) for every i with pred(i), pos = its rank among the flagged ones (index
// order); returns the count.  sh: kW + 1 ints.
template <typename Pred, typename Emit>
__device__ int cta_compact(int n, Pred pred, Emit emit, int* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int total = 0;
  for (int base = 0; base < n; base += kT) {
    const int i = base + threadIdx.x;
    const bool f = i < n && pred(i);
    const unsigned ball = __ballot_sync(LFPS_FULL, f);
    if (lane == 0) sh[warp] = __popc(ball);
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int w = 0; w < kW; ++w) {
        const int c = sh[w];
        sh[w] = acc;
        acc += c;
      }
      sh[kW] = acc;
    }
    __syncthreads();
    if (f) emit(total + sh[warp] + __popc(ball & ((1u << lane) - 1u)), i);
    total += sh[kW];
    __syncthreads();
  }
  return total;
}

// ---- row_logits (numerics.py:33-49): dot first, then / sqrt(d) ---------------
__global__ void stage_logits_kernel(const double* keys, int d, const int64_t* rows, int nrows,
                                    const double* q, double* out) {
  const int lane = threadIdx.x & 31;
  const int wid = (blockIdx.x * kT + threadIdx.x) >> 5;
  const int nw = (gridDim.x * kT) >> 5;
  const double sd = sqrt((double)d);
  for (int i = wid; i < nrows; i += nw) {
    const int64_t r = rows ? rows[i] : i;
    const double v = gdot_warp(keys + (size_t)r * d, q, d, lane);
    if (lane == 0) out[i] = cdiv(v, sd);
  }
}

// ---- compute_thresholds (tables.py:295-317) / thresholds_oracle (320-331) ----
// block t = table (0 vertical, 1 slash); 128 threads.  Canonical moments of
// x[0, m) (x = phys, or phys * scale when `materialize`): 512-slot segment
// moments, then the 512-leaf pairwise merge tree -- maintain_table's A and B
// over a window starting at slot 0.  out[3 t + {0,1,2}] = tau, mean,
// degenerate; out[6] = 3 when kappa == 0 (the ZeroDivisionError of
// tables.py:315).
__global__ void __launch_bounds__(128) stage_thresholds_kernel(const double* ver, const double* sla,
                                                              int m, double scale, double a,
                                                              int materialize, double* out,
                                                              double* scratch) {
  __shared__ tbl::Mom part[4];
  const int t = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* row = t ? sla : ver;
  const tbl::Window w = tbl::make_window(0, m);
  double* bs = scratch + (size_t)t * 4 * tbl::kLeaves;
  for (int blk = warp; blk < w.nseg; blk += 4) {
    int s0, vc;
    tbl::segment(w, blk, s0, vc);
    double v[16];
    tbl::load_seg(row, s0, vc, lane, v);
    if (materialize) {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = cmul(v[e], scale);
    }
    double mu, m2, m3, m4;
    if (vc == kBlk) tbl::seg_moments<true>(v, vc, lane, mu, m2, m3, m4);
    else tbl::seg_moments<false>(v, vc, lane, mu, m2, m3, m4);
    if (lane == 0) {
      double2* p = reinterpret_cast<double2*>(bs + 4 * (size_t)blk);
      p[0] = make_double2(mu, m2);
      p[1] = make_double2(m3, m4);
    }
  }
  __syncthreads();
  const tbl::Mom q = tbl::quarter_merge(bs, w, warp, lane);
  if (lane == 0) part[warp] = q;
  __syncthreads();
  if (threadIdx.x == 0) {
    const tbl::Mom tot = tbl::merge(tbl::merge(part[0], part[1]), tbl::merge(part[2], part[3]));
    const double sc = materialize ? 1.0 : scale;
    const double mean = cmul(tot.mu, sc);
    const bool deg = cmul(cmul(tot.m2, sc), sc) < 1e-12;
    double tau = NAN;
    if (!deg) {
      const double kappa = cdiv(tot.m4, cmul(tot.m2, tot.m2));
      if (kappa == 0.0) out[6] = 3.0;
      tau = cdiv(cmul(a, mean), kappa);
    }
    out[3 * t + 0] = tau;
    out[3 * t + 1] = mean;
    out[3 * t + 2] = deg ? 1.0 : 0.0;
  }
}

// ---- the three candidate stages (candidates.py:45-100), one CTA -------------
// mode 0 select_initial: slot i in C0 iff (!deg_v and ver[i] > tau_v / scale)
//        or (!deg_s and sla[i] > tau_s / scale);
// mode 1 expand: the in-range i + delta of every C0 entry, kept iff
//        ver[j] > mean_v / scale or sla[j] > mean_s / scale;
// mode 2 finalize_probe_set: C1 united with [max(S, n - L), n).
// Sets are sorted unique absolute indices (logical + base_index); the
// bitmap of the universe ([0, m) slots, or [0, n) positions) is in shared
// memory.
__global__ void stage_candidates_kernel(int mode, const double* ver, const double* sla, int m,
                                        double scale, const double* thr, const int64_t* in_idx,
                                        int n_in, const int* offsets, int n_off,
                                        long long base_index, int n, int sink, int window,
                                        int64_t* out_idx, int* out_count) {
  extern __shared__ uint32_t bits[];
  __shared__ int sh[kW + 1];
  const int U = mode == 2 ? n : m;                  // universe size
  const int words = (U + 31) / 32;
  if (mode == 0) {
    const bool dv = thr[2] != 0.0, ds = thr[5] != 0.0;
    const double tv = cdiv(thr[0], scale), ts = cdiv(thr[3], scale);
    const int cnt = cta_compact(
        m, [&](int i) { return (!dv && ver[i] > tv) || (!ds && sla[i] > ts); },
        [&](int pos, int i) { out_idx[pos] = i + base_index; }, sh);
    if (threadIdx.x == 0) *out_count = cnt;
    return;
  }
  for (int i = threadIdx.x; i < words; i += kT) bits[i] = 0u;
  __syncthreads();
  if (mode == 1) {
    for (int e = threadIdx.x; e < n_in * n_off; e += kT) {
      const long long j = in_idx[e / n_off] - base_index + offsets[e % n_off];
      if (j >= 0 && j < m) atomicOr(&bits[j >> 5], 1u << (j & 31));
    }
  } else {
    for (int e = threadIdx.x; e < n_in; e += kT) {
      const long long j = in_idx[e];
      if (j >= 0 && j < n) atomicOr(&bits[j >> 5], 1u << (j & 31));
    }
    const int lo = max(sink, n - window);
    for (int j = lo + threadIdx.x; j < n; j += kT) atomicOr(&bits[j >> 5], 1u << (j & 31));
  }
  __syncthreads();
  const double mv = mode == 1 ? cdiv(thr[1], scale) : 0.0;
  const double ms = mode == 1 ? cdiv(thr[4], scale) : 0.0;
  const long long off = mode == 1 ? base_index : 0;
  const int cnt = cta_compact(
      U,
      [&](int j) {
        if (!((bits[j >> 5] >> (j & 31)) & 1u)) return false;
        return mode == 2 || ver[j] > mv || sla[j] > ms;
      },
      [&](int pos, int j) { out_idx[pos] = j + off; }, sh);
  if (threadIdx.x == 0) *out_count = cnt;
}

// ---- topk_from_scores (attention.py:34-47): Top-k with lower-index ties ----
// idx ascending, scores aligned (fp64); k < p.  8 radix passes of 8 bits over
// an order-preserving 64-bit key find the k-th largest key; the output is
// every entry above it plus the lowest-index entries equal to it, ascending.
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
  if (u == 0x8000000000000000ull) u = 0ull;          // -0.0 ties +0.0
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

__global__ void stage_topk_kernel(const int64_t* idx, const double* scores, int p, int k,
                                  int64_t* out_idx, int* out_count) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long prefix_sh;
  __shared__ int want_sh, cut_sh;
  __shared__ int sh[kW + 1];
  if (k >= p) {                                     // pass-through (attention.py:39-40)
    for (int i = threadIdx.x; i < p; i += kT) out_idx[i] = idx[i];
    if (threadIdx.x == 0) *out_count = p;
    return;
  }
  unsigned long long prefix = 0ull, mask = 0ull;
  int want = k;                                     // rank of the k-th largest within the prefix
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int b = threadIdx.x; b < 256; b += kT) hist[b] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < p; i += kT) {
      const unsigned long long key = dkey(scores[i]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0, b = 255;
      for (; b > 0; --b) {
        if (acc + (int)hist[b] >= want) break;
        acc += hist[b];
      }
      want_sh = want - acc;
      prefix_sh = prefix | ((unsigned long long)b << shift);
    }
    __syncthreads();
    want = want_sh;
    prefix = prefix_sh;
    mask |= 255ull << shift;
    __syncthreads();
  }
  const unsigned long long kth = prefix;
  // `want` entries equal to kth are taken: the lowest-index ones; find the
  // position of the want-th equal entry, then one ordered compaction
  if (threadIdx.x == 0) cut_sh = p;
  __syncthreads();
  {
    int seen = 0;
    for (int base = 0; base < p; base += kT) {
      const int i = base + threadIdx.x;
      const bool eq = i < p && dkey(scores[i]) == kth;
      const unsigned ball = __ballot_sync(LFPS_FULL, eq);
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      if (lane == 0) sh[warp] = __popc(ball);
      __syncthreads();
      if (threadIdx.x == 0) {
        int acc = 0;
        for (int w = 0; w < kW; ++w) { const int c = sh[w]; sh[w] = acc; acc += c; }
        sh[kW] = acc;
      }
      __syncthreads();
      if (eq && seen + sh[warp] + __popc(ball & ((1u << lane) - 1u)) == want - 1) cut_sh = i;
      seen += sh[kW];
      __syncthreads();
      if (seen >= want) break;
    }
  }
  __syncthreads();
  const int cut = cut_sh;
  const int cnt = cta_compact(
      p, [&](int i) { const unsigned long long key = dkey(scores[i]);
                      return key > kth || (key == kth && i <= cut); },
      [&](int pos, int i) { out_idx[pos] = idx[i]; }, sh);
  if (threadIdx.x == 0) *out_count = cnt;
}

// ---- attention_output (attention.py:66-85) / full_attention_oracle (88-97) --
// logits over idx, max-shifted softmax (fp64 exp), out = w @ V[idx] with the
// weighted sum in ascending index order.  weights [nidx] doubles as the
// logit scratch; err = 7 on non-finite logits (numerics.py:61-62).
__global__ void stage_attend_kernel(const double* keys, const double* values, int d,
                                    const int64_t* idx, int nidx, const double* q, double* out,
                                    double* weights, int* err) {
  __shared__ double red[16];
  __shared__ int bad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double sd = sqrt((double)d);
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int i = warp; i < nidx; i += kW) {
    const int64_t r = idx ? idx[i] : i;
    const double v = cdiv(gdot_warp(keys + (size_t)r * d, q, d, lane), sd);
    if (lane == 0) {
      weights[i] = v;
      if (!isfinite(v)) bad = 1;
    }
  }
  __syncthreads();
  if (bad) {
    if (threadIdx.x == 0) *err = 7;
    return;
  }
  double mx = -INFINITY;
  for (int i = threadIdx.x; i < nidx; i += kT) mx = fmax(mx, weights[i]);
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(LFPS_FULL, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < kW; ++w) mx = fmax(mx, red[w]);
  __syncthreads();
  double acc = 0.0;
  for (int i = threadIdx.x; i < nidx; i += kT) {
    const double e = exp(csub(weights[i], mx));
    weights[i] = e;
    acc = cadd(acc, e);
  }
  const double tot = block_fold256(acc, red);
  for (int i = threadIdx.x; i < nidx; i += kT) weights[i] = cdiv(weights[i], tot);
  __syncthreads();
  for (int j = threadIdx.x; j < d; j += kT) {
    double o = 0.0;
    for (int i = 0; i < nidx; ++i) {
      const int64_t r = idx ? idx[i] : i;
      o = cadd(o, cmul(weights[i], values[(size_t)r * d + j]));
    }
    out[j] = o;
  }
  if (threadIdx.x == 0) *err = 0;
}

// ---- ScoreTablePair.update (tables.py:144-200), after the host's checks ----
// sla points at the slash buffer, base = the window start before this
// update's shift.  renorm: renormalisation by rf first (vertical [0, m),
// slash [base, base + m], tables.py:240-244).  Then the shift (slot base - 1
// zeroed), add = (w - 1 / (2k)) / scale folded into ver[sel] and
// sla[base - 1 + sel] with numpy fancy-index semantics (reads, then writes in
// order), negatives clamped to 0 and counted into *clamps.
__global__ void stage_update_kernel(double* ver, double* sla, int base, int m, const int64_t* sel,
                                    const double* w, int k, int renorm, double rf, double scale,
                                    long long* clamps, double* tmp) {
  __shared__ double red[16];
  const int tid = threadIdx.x;
  if (renorm) {
    for (int i = tid; i < m; i += kT) ver[i] = cmul(ver[i], rf);
    for (int i = tid; i <= m; i += kT) sla[base + i] = cmul(sla[base + i], rf);
    __syncthreads();
  }
  const int nb = base - 1;
  if (tid == 0) sla[nb] = 0.0;
  __syncthreads();
  const double inv = cdiv(1.0, cmul(2.0, (double)k));
  long long nneg = 0;
  for (int pass = 0; pass < 2; ++pass) {
    double* tab = pass ? sla + nb : ver;
    for (int i = tid; i < k; i += kT) tmp[i] = cadd(tab[sel[i]], cdiv(csub(w[i], inv), scale));
    __syncthreads();
    if (tid == 0)
      for (int i = 0; i < k; ++i) tab[sel[i]] = tmp[i];
    __syncthreads();
    for (int i = tid; i < k; i += kT) tmp[i] = tab[sel[i]];
    __syncthreads();
    for (int i = tid; i < k; i += kT)
      if (tmp[i] < 0.0) { ++nneg; tab[sel[i]] = 0.0; }
    __syncthreads();
  }
  const double tot = block_fold256((double)nneg, red);
  if (tid == 0) *clamps = (long long)tot;
}

// ---- ScoreTablePair.grow (tables.py:202-220) --------------------------------
__global__ void stage_grow_kernel(double* ver, double* sla, int base, int m, int carry) {
  ver[m] = 0.0;
  if (!carry) sla[base + m] = 0.0;
}

// ---- init_tables (tables.py:247-281): Eq. 4 seeding --------------------------
// column sums (rows oldest first, numpy's axis-0 order) and diagonal sums,
// times 1 / (2 s (1 - r)); multi-CTA, one slot per thread
__global__ void stage_init_tables_kernel(const double* w, int s, int m, double r, double* ver,
                                         double* sla) {
  const double coeff = cdiv(1.0, cmul(cmul(2.0, (double)s), csub(1.0, r)));
  for (int i = blockIdx.x * kT + threadIdx.x; i < m; i += gridDim.x * kT) {
    double cv = 0.0, cs = 0.0;
    for (int c = 0; c < s; ++c) {
      cv = cadd(cv, w[(size_t)c * m + i]);
      const int off = s - c - 1;
      if (off < m && i >= off) cs = cadd(cs, w[(size_t)c * m + i - off]);
    }
    ver[i] = cmul(cv, coeff);
    sla[i] = cmul(cs, coeff);
  }
}

// ---- compute_head_stats (gate.py:51-74) --------------------------------------
// mean key / value over rows [S, n) (sequential per column, numpy's axis-0
// order), sigma^2 = var(logits of the last prefill query) / |q|^2 with the
// logits in the canonical dot order; err = 6 on a zero-norm query.
__global__ void stage_head_stats_kernel(const double* keys, const double* values, int n, int d,
                                        int sink, const double* q, double* mean_key,
                                        double* mean_value, double* sigma, double* logit_tmp,
                                        int* err) {
  __shared__ double red[16];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cnt = n - sink;
  for (int j = threadIdx.x; j < d; j += kT) {
    double sk = 0.0, sv = 0.0;
    for (int i = sink; i < n; ++i) {
      sk = cadd(sk, keys[(size_t)i * d + j]);
      sv = cadd(sv, values[(size_t)i * d + j]);
    }
    mean_key[j] = cdiv(sk, (double)cnt);
    mean_value[j] = cdiv(sv, (double)cnt);
  }
  const double sd = sqrt((double)d);
  for (int i = warp; i < cnt; i += kW) {
    const double v = cdiv(gdot_warp(keys + (size_t)(sink + i) * d, q, d, lane), sd);
    if (lane == 0) logit_tmp[i] = v;
  }
  const double qq = gdot_warp(q, q, d, lane);
  __syncthreads();
  double acc = 0.0;
  for (int i = threadIdx.x; i < cnt; i += kT) acc = cadd(acc, logit_tmp[i]);
  const double mu = cdiv(block_fold256(acc, red), (double)cnt);
  acc = 0.0;
  for (int i = threadIdx.x; i < cnt; i += kT) {
    const double dv = csub(logit_tmp[i], mu);
    acc = cadd(acc, cmul(dv, dv));
  }
  const double var = cdiv(block_fold256(acc, red), (double)cnt);
  if (threadIdx.x == 0) {
    *err = qq == 0.0 ? 6 : 0;
    *sigma = cdiv(var, qq);
  }
}

// ---- gate (gate.py:77-147): logits, sparsity estimate, bypass output -------
// out: [S] sink logits, [L] local logits (rows [n - L, n)), gexp, w_sink,
// w_global, w_local, rho, then the bypass output [d] (bypass_mode 1:
// mean_only, 0: sink_average).  err = 1 non-finite logits, 2 non-finite rho.
__global__ void stage_gate_kernel(const double* keys, const double* values, int n, int d, int sink,
                                  int window, const double* q, const double* mean_key,
                                  const double* mean_value, double sigma, int bypass_mode,
                                  double* out, int* err) {
  __shared__ double lg[64 + 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double sd = sqrt((double)d);
  const int nl = sink + window;
  for (int i = warp; i < nl + 2; i += kW) {
    double v;
    if (i < sink) v = cdiv(gdot_warp(keys + (size_t)i * d, q, d, lane), sd);
    else if (i < nl) v = cdiv(gdot_warp(keys + (size_t)(n - window + i - sink) * d, q, d, lane), sd);
    else if (i == nl) v = gdot_warp(q, mean_key, d, lane);   // q . K-bar
    else v = gdot_warp(q, q, d, lane);                       // |q|^2
    if (lane == 0) lg[i] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // global_exponent (gate.py:77-81): q.K-bar / sqrt(d) + |q|^2 sigma / 2
    const double g = cadd(cdiv(lg[nl], sd), cdiv(cmul(lg[nl + 1], sigma), 2.0));
    bool fin = isfinite(g);
    double shift = g;
    for (int i = 0; i < nl; ++i) {
      fin = fin && isfinite(lg[i]);
      shift = fmax(shift, lg[i]);
    }
    int e = 0;
    double ws = 0.0, wl = 0.0, wg = 0.0, rho = NAN;
    if (!fin) {
      e = 1;
    } else {
      for (int i = 0; i < sink; ++i) ws = cadd(ws, exp(csub(lg[i], shift)));
      for (int i = sink; i < nl; ++i) wl = cadd(wl, exp(csub(lg[i], shift)));
      wg = cmul(exp(csub(g, shift)), (double)(n - sink));
      rho = cdiv(ws, cadd(cadd(ws, wg), wl));
      if (!isfinite(rho)) e = 2;
    }
    for (int i = 0; i < nl; ++i) out[i] = lg[i];
    out[nl] = g;
    out[nl + 1] = ws;
    out[nl + 2] = wg;
    out[nl + 3] = wl;
    out[nl + 4] = rho;
    lg[nl] = g;
    *err = e;
  }
  __syncthreads();
  // bypass_output (gate.py:131-147)
  double* bo = out + nl + 5;
  if (bypass_mode == 1) {
    for (int j = threadIdx.x; j < d; j += kT) bo[j] = mean_value[j];
    return;
  }
  // softmax over [sink logits..., gexp]
  double mx = lg[nl];
  for (int i = 0; i < sink; ++i) mx = fmax(mx, lg[i]);
  double tot = 0.0;
  for (int i = 0; i < sink; ++i) tot = cadd(tot, exp(csub(lg[i], mx)));
  tot = cadd(tot, exp(csub(lg[nl], mx)));
  for (int j = threadIdx.x; j < d; j += kT) {
    double o = 0.0;
    for (int i = 0; i < sink; ++i)
      o = cadd(o, cmul(cdiv(exp(csub(lg[i], mx)), tot), values[(size_t)i * d + j]));
    bo[j] = cadd(o, cmul(cdiv(exp(csub(lg[nl], mx)), tot), mean_value[j]));
  }
}

}  // namespace

cudaError_t stage_logits(const double* keys, int d, const int64_t* rows, int nrows, const double* q,
                         double* out, cudaStream_t st) {
  const int blocks = nrows < 1 ? 1 : (nrows + kW - 1) / kW < 1184 ? (nrows + kW - 1) / kW : 1184;
  stage_logits_kernel<<<blocks, kT, 0, st>>>(keys, d, rows, nrows, q, out);
  return cudaGetLastError();
}

cudaError_t stage_thresholds(const double* ver, const double* sla, int m, double scale, double a,
                             int materialize, double* out, double* scratch, cudaStream_t st) {
  stage_thresholds_kernel<<<2, 128, 0, st>>>(ver, sla, m, scale, a, materialize, out, scratch);
  return cudaGetLastError();
}

cudaError_t stage_candidates(int mode, const double* ver, const double* sla, int m, double scale,
                             const double* thr, const int64_t* in_idx, int n_in, const int* offsets,
                             int n_off, long long base_index, int n, int sink, int window,
                             int64_t* out_idx, int* out_count, cudaStream_t st) {
  const int U = mode == 2 ? n : m;
  const size_t smem = mode == 0 ? 0 : (size_t)((U + 31) / 32) * 4;
  static DeviceOnce once;
  cudaError_t e = once.run([] {
    return cudaFuncSetAttribute(stage_candidates_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                200 * 1024);
  });
  if (e != cudaSuccess) return e;
  stage_candidates_kernel<<<1, kT, smem, st>>>(mode, ver, sla, m, scale, thr, in_idx, n_in, offsets,
                                               n_off, base_index, n, sink, window, out_idx,
                                               out_count);
  return cudaGetLastError();
}

cudaError_t stage_topk(const int64_t* idx, const double* scores, int p, int k, int64_t* out_idx,
                       int* out_count, cudaStream_t st) {
  stage_topk_kernel<<<1, kT, 0, st>>>(idx, scores, p, k, out_idx, out_count);
  return cudaGetLastError();
}

cudaError_t stage_attend(const double* keys, const double* values, int d, const int64_t* idx,
                         int nidx, const double* q, double* out, double* weights, int* err,
                         cudaStream_t st) {
  stage_attend_kernel<<<1, kT, 0, st>>>(keys, values, d, idx, nidx, q, out, weights, err);
  return cudaGetLastError();
}

cudaError_t stage_update(double* ver, double* sla, int base, int m, const int64_t* sel,
                         const double* w, int k, int renorm, double rf, double scale,
                         long long* clamps, double* tmp, cudaStream_t st) {
  stage_update_kernel<<<1, kT, 0, st>>>(ver, sla, base, m, sel, w, k, renorm, rf, scale, clamps,
                                        tmp);
  return cudaGetLastError();
}

cudaError_t stage_grow(double* ver, double* sla, int base, int m, int carry, cudaStream_t st) {
  stage_grow_kernel<<<1, 1, 0, st>>>(ver, sla, base, m, carry);
  return cudaGetLastError();
}

cudaError_t stage_init_tables(const double* w, int s, int m, double r, double* ver, double* sla,
                              cudaStream_t st) {
  int blocks = (m + kT - 1) / kT;
  if (blocks > 1184) blocks = 1184;
  stage_init_tables_kernel<<<blocks, kT, 0, st>>>(w, s, m, r, ver, sla);
  return cudaGetLastError();
}

cudaError_t stage_head_stats(const double* keys, const double* values, int n, int d, int sink,
                             const double* q, double* mean_key, double* mean_value, double* sigma,
                             double* logit_tmp, int* err, cudaStream_t st) {
  stage_head_stats_kernel<<<1, kT, 0, st>>>(keys, values, n, d, sink, q, mean_key, mean_value,
                                            sigma, logit_tmp, err);
  return cudaGetLastError();
}

cudaError_t stage_gate(const double* keys, const double* values, int n, int d, int sink, int window,
                       const double* q, const double* mean_key, const double* mean_value,
                       double sigma, int bypass_mode, double* out, int* err, cudaStream_t st) {
  stage_gate_kernel<<<1, kT, 0, st>>>(keys, values, n, d, sink, window, q, mean_key, mean_value,
                                      sigma, bypass_mode, out, err);
  return cudaGetLastError();
}

}  // namespace lfps
