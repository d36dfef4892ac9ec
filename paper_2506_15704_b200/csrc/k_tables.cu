// k_tables.cu -- tracker tables -> thresholds -> C0 candidates, ONE table read.
//
// Restates compute_thresholds (tables.py:295-317) and select_initial
// (candidates.py:45-58) for every (session, table) item of the batch.
//
//   lfps_stats_kernel    streams every table once (coalesced 8-byte lane loads,
//                   no inter-CTA synchronisation): per 512-slot chunk the
//                   mean and centred power sums M2, M3, M4 (canonical
//                   devmath.chunk_moments), and a capture of every slot whose
//                   phys value exceeds the item's capture bound L (index and
//                   value appended to a per-item list).
//   lfps_thresh_kernel   one warp per item: merges the chunk moments (exact
//                   pairwise updates, canonical tree) into mean, s2, s4 and
//                   derives tau/scale, mean/scale and the degenerate flag.
//                   C0 = {slots with phys > tau/scale}; because the capture
//                   bound satisfies L <= tau/scale, every member of C0 is in
//                   the capture list, so C0 is decided exactly (fp64 compare)
//                   without a second pass over the table.  If that guarantee
//                   fails (no bound yet, bound above tau/scale, or the list
//                   overflowed) the item is queued for the fallback.
//   lfps_fallback_kernel rare: re-reads a queued item and writes its C0 bitmap.
//
// The capture bound is half of the item's previous-step tau/scale: between
// steps the lazy scale only shrinks (r < 1), so tau/scale in phys units grows
// and the bound stays valid; a renormalisation or a first step simply takes
// the fallback.  HBM traffic is the tables once plus the (small) captures.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 512;
constexpr int kLeaves = 512;                 // chunks per table: m <= 262144
constexpr int kLeavesPerLane = kLeaves / 32;

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

// phys slot of logical index i of an item (ver: i; sla: ring)
__device__ __forceinline__ const double* item_row(const Ctx& c, int item) {
  const int s = item >> 1;
  return (item & 1) ? c.sla + (size_t)s * c.ring_cap : c.ver + (size_t)s * c.m_cap;
}

// 16 slots of chunk ch for this lane (logical ch*512 + e*32 + lane), 0 if >= m
__device__ __forceinline__ void load_chunk(const Ctx& c, int item, int base, int m, int ch,
                                           int lane, double* v) {
  const double* row = item_row(c, item);
  const int i0 = ch * kChunk;
  if ((item & 1) == 0) {
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = i0 + e * 32 + lane;
      v[e] = i < m ? __ldcs(row + i) : 0.0;
    }
  } else {
    const int C = c.ring_cap;
    const int p0 = (base + i0) % C;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = i0 + e * 32 + lane;
      int p = p0 + e * 32 + lane;
      if (p >= C) p -= C;
      v[e] = i < m ? __ldcs(row + p) : 0.0;
    }
  }
}

// chunk moments of 16 lane values (v beyond the valid count vc are 0);
// FULL: all 512 slots valid (no masking)
template <bool FULL>
__device__ __forceinline__ void chunk_moments(const double* v, int vc, int lane, double& mu,
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

// ---------------------------------------------------------------------------
// lfps_stats_kernel: one warp per (item, chunk), grid-stride
// ---------------------------------------------------------------------------
struct ChunkRef {
  int item, ch, m, vc, base;
  bool live;
};

__device__ __forceinline__ void chunk_process(const Ctx& c, const ChunkRef& r, const double* v,
                                              int lane) {
  double mu, m2, m3, m4;
  if (r.vc == kChunk) chunk_moments<true>(v, r.vc, lane, mu, m2, m3, m4);
  else chunk_moments<false>(v, r.vc, lane, mu, m2, m3, m4);
  double* cs = c.tb.cstat + ((size_t)r.item * kLeaves + r.ch) * 4;
  if (lane == 0) {
    cs[0] = mu; cs[1] = m2; cs[2] = m3; cs[3] = m4;
  }
  // capture slots above the bound (index + value)
  const double L = c.tb.bound[r.item];
  if (L > 0.0) {
    const long long Lb = __double_as_longlong(L);
    // early out: most chunks hold nothing above the bound (invalid slots are 0)
    long long mx = __double_as_longlong(v[0]);
#pragma unroll
    for (int e = 1; e < 16; ++e) mx = max(mx, __double_as_longlong(v[e]));
    if (!__any_sync(LFPS_FULL, mx > Lb)) return;
    int nmy = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) nmy += (__double_as_longlong(v[e]) > Lb) && (e * 32 + lane < r.vc);
    int incl = nmy;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(LFPS_FULL, incl, o);
      if (lane >= o) incl += y;
    }
    const int tot = __shfl_sync(LFPS_FULL, incl, 31);
    if (tot > 0) {
      int at = 0;
      if (lane == 31) at = atomicAdd(c.tb.ncap + r.item, tot);
      at = __shfl_sync(LFPS_FULL, at, 31) + incl - nmy;
      int* ci = c.tb.cidx + (size_t)r.item * c.tb.cap;
      double* cv = c.tb.cval + (size_t)r.item * c.tb.cap;
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int i = r.ch * kChunk + e * 32 + lane;
        if ((__double_as_longlong(v[e]) > Lb) && (e * 32 + lane < r.vc)) {
          if (at < c.tb.cap) {
            ci[at] = i;
            cv[at] = v[e];
          }
          ++at;
        }
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 3) lfps_stats_kernel(Ctx c, int nch_max) {
  const int lane = threadIdx.x & 31;
  const int n_items = 2 * c.NS;
  const int stride = gridDim.x * kWarps;
  const int q = stride / nch_max, rem = stride % nch_max;
  const int w0 = blockIdx.x * kWarps + (threadIdx.x >> 5);
  int item = w0 / nch_max, ch = w0 % nch_max;
  for (; item < n_items; item += q, ch += rem) {
    if (ch >= nch_max) { ch -= nch_max; ++item; if (item >= n_items) break; }
    const int s = item >> 1;
    const int m = c.n_ctx[s / c.Hq] - c.S;
    if (ch * kChunk >= m || c.bypass[s]) continue;
    ChunkRef r;
    r.item = item;
    r.ch = ch;
    r.m = m;
    r.vc = min(kChunk, m - ch * kChunk);
    r.base = (item & 1) ? c.sla_base[s] : 0;
    r.live = true;
    double v[16];
    load_chunk(c, r.item, r.base, r.m, r.ch, lane, v);
    chunk_process(c, r, v, lane);
  }
}

// ---------------------------------------------------------------------------
// lfps_thresh_kernel: one warp per item
// ---------------------------------------------------------------------------
__device__ __noinline__ Mom item_merge(const double* cs, int n_chunks, int m, int lane) {
  Mom stk[4];
  Mom cur;
#pragma unroll
  for (int k = 0; k < kLeavesPerLane; ++k) {
    const int i = lane * kLeavesPerLane + k;
    cur = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (i < n_chunks) {
      cur.n = (double)min(kChunk, m - i * kChunk);
      const double4 q = *reinterpret_cast<const double4*>(cs + 4 * i);
      cur.mu = q.x; cur.m2 = q.y; cur.m3 = q.z; cur.m4 = q.w;
    }
#pragma unroll
    for (int l = 0; l < 4; ++l) {
      if ((k >> l) & 1) {
        cur = merge(stk[l], cur);
      } else {
        stk[l] = cur;
        break;
      }
    }
  }
  Mom acc = cur;
#pragma unroll
  for (int h = 1; h <= 16; h <<= 1) {
    const Mom o = shfl_mom(acc, h);
    acc = (lane & h) ? merge(o, acc) : merge(acc, o);
  }
  return acc;
}

__global__ void __launch_bounds__(kThreads) lfps_thresh_kernel(Ctx c) {
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (item >= 2 * c.NS) return;
  const int s = item >> 1;
  double* itf = c.tb.itemf + (size_t)item * 4;
  if (c.bypass[s]) return;
  const int m = c.n_ctx[s / c.Hq] - c.S;
  const double sc = c.scale[s];
  double* thr = c.thr + (size_t)item * 4;
  if (c.exhaustive) {
    if (lane == 0) {
      itf[0] = -INFINITY; itf[1] = -INFINITY; itf[2] = 0.0;
      thr[0] = -INFINITY; thr[1] = -INFINITY; thr[2] = 0.0; thr[3] = NAN;
    }
    return;
  }
  const Mom tot = item_merge(c.tb.cstat + (size_t)item * kLeaves * 4, (m + kChunk - 1) / kChunk,
                             m, lane);
  if (lane != 0) return;
  const double mean = cmul(tot.mu, sc);
  const bool deg = cmul(cmul(tot.m2, sc), sc) < 1e-12;
  double tau = NAN, kappa = NAN, thr0 = NAN;
  if (!deg) {
    kappa = cdiv(tot.m4, cmul(tot.m2, tot.m2));
    if (kappa == 0.0) set_err(c, s, LFPS_ERR_KAPPA_ZERO);
    tau = cdiv(cmul(c.a, mean), kappa);
    thr0 = cdiv(tau, sc);
  }
  itf[0] = thr0;
  itf[1] = cdiv(mean, sc);
  itf[2] = deg ? 1.0 : 0.0;
  thr[0] = tau; thr[1] = mean; thr[2] = deg ? 1.0 : 0.0; thr[3] = kappa;
  // was every C0 member captured?  (C0 empty when degenerate or thr0 is NaN / +inf)
  const double L = c.tb.bound[item];
  const bool empty_c0 = deg || !(thr0 < INFINITY);
  const bool ok = empty_c0 || (L > 0.0 && L <= thr0 && c.tb.ncap[item] <= c.tb.cap);
  c.tb.fb[item] = ok ? 0 : 1;
  if (!ok) {
    const int q = atomicAdd(c.tb.nfb, 1);
    c.tb.fblist[q] = item;
  }
  // capture bound for the next step: half of this step's tau/scale
  c.tb.bound[item] = (!deg && thr0 > 0.0 && thr0 < INFINITY) ? cmul(thr0, 0.5) : 0.0;
}

// ---------------------------------------------------------------------------
// lfps_fallback_kernel: C0 bitmap of queued items (one warp per chunk)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) lfps_fallback_kernel(Ctx c, int nch_max) {
  const int lane = threadIdx.x & 31;
  const int nq = *c.tb.nfb;
  const long long n_work = (long long)nq * nch_max;
  const long long wstride = (long long)gridDim.x * kWarps;
  for (long long w = (long long)blockIdx.x * kWarps + (threadIdx.x >> 5); w < n_work; w += wstride) {
    const int item = c.tb.fblist[w / nch_max];
    const int ch = (int)(w % nch_max);
    const int s = item >> 1;
    const int m = c.n_ctx[s / c.Hq] - c.S;
    if (ch * kChunk >= m) continue;
    const int base = (item & 1) ? c.sla_base[s] : 0;
    double v[16];
    load_chunk(c, item, base, m, ch, lane, v);
    const long long tb = __double_as_longlong(c.tb.itemf[(size_t)item * 4]);  // thr0 >= 0
    uint32_t my = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const bool ok = ch * kChunk + e * 32 + lane < m;
      const uint32_t wd = __ballot_sync(LFPS_FULL, ok && __double_as_longlong(v[e]) > tb);
      if (lane == e) my = wd;
    }
    if (lane < 16) c.bits[(size_t)item * c.words + ch * 16 + lane] = my;
  }
}

__global__ void lfps_tables_reset_kernel(Ctx c) {
  const int n = 2 * c.NS;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    c.tb.ncap[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *c.tb.nfb = 0;
}

int g_stats_grid = 0;

}  // namespace

cudaError_t launch_tables(const Ctx& c, int m_max, cudaStream_t st) {
  const int nch_max = (m_max + kChunk - 1) / kChunk;
  if (nch_max > kLeaves) return cudaErrorInvalidValue;
  if (!g_stats_grid) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lfps_stats_kernel, kThreads, 0);
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_stats_grid = sms * (per_sm > 0 ? per_sm : 1);
  }
  lfps_tables_reset_kernel<<<16, 256, 0, st>>>(c);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  if (!c.exhaustive) {
    const long long work = (long long)2 * c.NS * nch_max;
    long long grid = (work + kWarps - 1) / kWarps;
    if (grid > g_stats_grid) grid = g_stats_grid;
    lfps_stats_kernel<<<(int)grid, kThreads, 0, st>>>(c, nch_max);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  lfps_thresh_kernel<<<(2 * c.NS + kWarps - 1) / kWarps, kThreads, 0, st>>>(c);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (!c.exhaustive) {
    lfps_fallback_kernel<<<g_stats_grid, kThreads, 0, st>>>(c, nch_max);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  return cudaSuccess;
}

int tables_launches(void) { return 4; }

}  // namespace lfps
