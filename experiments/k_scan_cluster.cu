// k_scan.cu -- tracker-table scan: moments + thresholds (K1) and the
// candidate bitmaps (first half of K2), one read of every table.
//
// Persistent thread-block clusters; cluster c walks the (session, table)
// items c, c + NC, c + 2 NC, ...  Each CTA of a cluster owns a contiguous
// slice of the item's logical range and keeps it in shared memory:
//
//   load    1-D bulk async copies (cp.async.bulk + mbarrier) of the slice,
//           served from L2: while item i is processed, the slice of item
//           i + NC was already requested with cp.async.bulk.prefetch.L2, so
//           HBM streams underneath the compute phases
//   stats   per 512-slot chunk: mean and centred power sums M2, M3, M4
//           (devmath.chunk_moments); each chunk's four values are sent
//           straight into the leader CTA's shared memory with st.async
//           (mbarrier complete_tx), no cluster barrier
//   merge   the leader merges all chunks of the table with exact pairwise
//           updates (devmath.merge_moments, canonical tree) into mean, s2,
//           s4, derives tau / mean / degenerate (tables.py:295-317) and
//           st.async-broadcasts the two thresholds to every CTA
//   bits    ballot bitmaps over the resident slice: C0 = phys > tau/scale
//           (select_initial, candidates.py:45-58), F = phys > mean/scale
//           (expand's filter, candidates.py:79-81), compared on the fp64 bit
//           patterns (all phys values are +0 or positive)
//
// The table is read from HBM exactly once; the two bitmaps written are 1/32
// of it.  Results are bit-identical to oracle/devmath.table_moments and
// independent of the cluster shape.
#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 384;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 512;          // canonical chunk (devmath.TABLE_CHUNK)
constexpr int kGroup = 8;            // chunks pre-merged inside a CTA (aligned subtree)
constexpr int kGroupSlots = kChunk * kGroup;   // 4096
constexpr int kStage = 1024;         // elements per bulk-copy stage (8 KB)
constexpr int kMaxStages = 16;
constexpr int kMaxSlice = 3 * kGroupSlots;     // 12288 slots = 96 KB per CTA
constexpr int kTreeLeaves = 64;      // >= groups of the largest supported table
constexpr int kLeavesPerLane = kTreeLeaves / 32;

struct Shared {
  uint64_t bar[kMaxStages];   // bulk-copy stages (one phase per item)
  uint64_t gat_bar[2];        // leader: group moments of the cluster landed (by item parity)
  uint64_t res_bar[2];        // every CTA: the leader's thresholds landed (by item parity)
  double bcast[2][4];         // thr0, thrf, deg (by item parity)
};

// chunk moments (count, mean, M2, M3, M4)
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

// Canonical merge tree over the gathered group moments g[i][0..3] (groups of
// 8 chunks are aligned subtrees of the chunk tree; zero-count padding to
// kTreeLeaves); lane l owns leaves 2l, 2l+1; all lanes return the total.
__device__ __forceinline__ Mom group_leaf(const double* g, int i, int n_groups, int m) {
  Mom r = {0.0, 0.0, 0.0, 0.0, 0.0};
  if (i < n_groups) {
    r.n = (double)min(kGroupSlots, m - i * kGroupSlots);
    r.mu = g[4 * i];
    r.m2 = g[4 * i + 1];
    r.m3 = g[4 * i + 2];
    r.m4 = g[4 * i + 3];
  }
  return r;
}

__device__ __noinline__ Mom merge_tree(const double* g, int n_groups, int m, int lane) {
  Mom acc = merge(group_leaf(g, 2 * lane, n_groups, m), group_leaf(g, 2 * lane + 1, n_groups, m));
#pragma unroll
  for (int h = 1; h <= 16; h <<= 1) {
    const Mom o = shfl_mom(acc, h);
    acc = (lane & h) ? merge(o, acc) : merge(acc, o);
  }
  return acc;
}

// Per-item metadata, loaded one item ahead so no dependent global-load chain
// sits on the critical path of an item's start.
struct Meta {
  int byp, m, base;
  double sc;
};
__device__ __forceinline__ Meta load_meta(const Ctx& c, int item, int n_items) {
  Meta t = {1, 0, 0, 1.0};
  if (item < n_items) {
    const int s = item >> 1;
    t.byp = c.bypass[s];
    t.m = c.n_ctx[s / c.Hq] - c.S;
    t.base = c.sla_base[s];
    t.sc = c.scale[s];
  }
  return t;
}

// Pieces of logical range [l0, l0 + len) of a table (ver: contiguous; sla:
// ring of C slots).  Returns the piece count (1-2).
struct Piece {
  const double* p;
  int n;
};
__device__ __forceinline__ int table_pieces(const Ctx& c, int s, int table, int base, int l0,
                                            int len, Piece* out) {
  if (table == 0) {
    out[0] = {c.ver + (size_t)s * c.m_cap + l0, len};
    return 1;
  }
  const int C = c.ring_cap;
  const double* ring = c.sla + (size_t)s * C;
  const int p = ((base + l0) % C + C) % C;
  const int first = min(len, C - p);
  out[0] = {ring + p, first};
  if (first < len) {
    out[1] = {ring, len - first};
    return 2;
  }
  return 1;
}

// smem element e <-> logical (lo - off + e); off keeps copies 16-B aligned
__device__ __forceinline__ int slice_off(const Ctx& c, int table, int base, int lo) {
  return table == 1 ? (((base + lo) % c.ring_cap) & 1) : 0;
}

__device__ __forceinline__ void prefetch_item(const Ctx& c, int item, const Meta& mt, int slice,
                                              uint32_t rank) {
  if (mt.byp || c.exhaustive) return;
  const int s = item >> 1, table = item & 1;
  const int lo = (int)rank * slice;
  const int cnt = max(0, min(slice, mt.m - lo));
  if (cnt == 0) return;
  const int off = slice_off(c, table, mt.base, lo);
  const int total = (off + cnt + 1) & ~1;
  Piece pc[2];
  const int np = table_pieces(c, s, table, mt.base, lo - off, total, pc);
  for (int k = 0; k < np; ++k) prefetch_l2(pc[k].p, (uint32_t)pc[k].n * 8u);
}

// fp64 bit pattern of a threshold for integer comparison against phys
// values (all phys values are +0.0 or positive finite, so for thr in
// [+0, +inf] the int64 order equals the IEEE order; NaN never compares true).
__device__ __forceinline__ long long thr_bits(double t) {
  return isnan(t) ? 0x7fffffffffffffffll : __double_as_longlong(t);
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One (session, table) item as this CTA sees it.
struct Item {
  int item, s, table, m, base, cnt, off;
  double sc;
};

__device__ __forceinline__ Item make_item(const Ctx& c, int item, int n_items, int slice, int lo) {
  Item it;
  it.item = item;
  if (item >= n_items) {
    it.s = it.table = it.m = it.base = it.cnt = it.off = 0;
    it.sc = 1.0;
    return it;
  }
  it.s = item >> 1;
  it.table = item & 1;
  it.m = c.n_ctx[it.s / c.Hq] - c.S;
  it.base = it.table ? c.sla_base[it.s] : 0;
  it.sc = c.scale[it.s];
  it.cnt = max(0, min(slice, it.m - lo));
  it.off = it.table ? (((it.base + lo) % c.ring_cap) & 1) : 0;
  return it;
}

// next non-bypassed item of this cluster's sequence at or after `item`
__device__ __forceinline__ int next_valid(const Ctx& c, int item, int n_items, int stride) {
  while (item < n_items && c.bypass[item >> 1]) item += stride;
  return item;
}

// warp 0: bulk copies of the item's slice into smem, one lane per stage
__device__ __forceinline__ void issue_copies(const Ctx& c, const Item& it, double* data,
                                             Shared* sh, int lo, int lane) {
  const int total = it.cnt > 0 ? ((it.off + it.cnt + 1) & ~1) : 0;   // even element count
  const int nst = (total + kStage - 1) / kStage;
  if (lane < kMaxStages) {
    const int j = lane;
    if (j < nst) {
      const int e0 = j * kStage;
      const int len = min(kStage, total - e0);
      mbar_expect_tx(&sh->bar[j], (uint32_t)len * 8u);
      Piece pc[2];
      const int np = table_pieces(c, it.s, it.table, it.base, lo - it.off + e0, len, pc);
      int at = e0;
      for (int k = 0; k < np; ++k) {
        bulk_g2s(data + at, pc[k].p, (uint32_t)pc[k].n * 8u, &sh->bar[j]);
        at += pc[k].n;
      }
    } else {
      mbar_arrive(&sh->bar[j]);             // keep every stage's phase in step
    }
  }
}

__device__ __forceinline__ void prefetch_slice(const Ctx& c, const Item& it, int lo) {
  if (it.cnt == 0) return;
  const int total = (it.off + it.cnt + 1) & ~1;
  Piece pc[2];
  const int np = table_pieces(c, it.s, it.table, it.base, lo - it.off, total, pc);
  for (int k = 0; k < np; ++k) prefetch_l2(pc[k].p, (uint32_t)pc[k].n * 8u);
}

// bitmaps of the CTA's slice of `it`, re-read from L2 (the smem copy already
// holds the next item)
__device__ __forceinline__ void slice_bits(const Ctx& c, const Item& it, int lo, int words_cta,
                                           long long tb0, long long tbf, int warp, int lane) {
  uint32_t* bits_c0 = c.bits + ((size_t)it.item * 2 + 0) * c.words;
  uint32_t* bits_f = c.bits + ((size_t)it.item * 2 + 1) * c.words;
  const int C = c.ring_cap;
  const long long* ver = reinterpret_cast<const long long*>(c.ver + (size_t)it.s * c.m_cap);
  const long long* ring = reinterpret_cast<const long long*>(c.sla + (size_t)it.s * C);
  for (int g0 = warp * 32; g0 < words_cta; g0 += kWarps * 32) {
    uint32_t my0 = 0, myf = 0;
    const int nw = min(32, words_cta - g0);
    const int i0 = g0 * 32;                  // CTA-local slot of the group's first word
    if (i0 < it.cnt) {
      const int p0 = it.table ? (it.base + lo + i0) % C : lo + i0;
      const long long* src = it.table ? ring : ver;
      // 16 independent L2 loads in flight per lane, then the ballots
#pragma unroll
      for (int jb = 0; jb < 32; jb += 16) {
        long long x[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int j = jb + t;
          int p = p0 + j * 32 + lane;
          if (it.table && p >= C) p -= C;
          const bool valid = j < nw && i0 + j * 32 + lane < it.cnt;
          x[t] = valid ? __ldcg(src + p) : -1ll;
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const uint32_t w0 = __ballot_sync(LFPS_FULL, x[t] > tb0);
          const uint32_t wf = __ballot_sync(LFPS_FULL, x[t] > tbf);
          if (lane == jb + t) { my0 = w0; myf = wf; }
        }
      }
    }
    if (lane < nw) {
      bits_c0[lo / 32 + g0 + lane] = my0;
      bits_f[lo / 32 + g0 + lane] = myf;
    }
  }
}

// MODE (experiments, tools/scan_bench.cu): 0 = production, 3 = production
// plus a per-phase globaltimer trace of cluster 0 written to c.scratch.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) scan_kernel(Ctx c, int slice, int n_items) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cs = (int)cluster_size();
  const int cpc = slice / kChunk;                // chunks per CTA
  const int gpc = slice / kGroupSlots;           // groups per CTA
  const int gsz = cs * gpc;                      // group leaves per table
  double* data = reinterpret_cast<double*>(smem_raw);                 // [slice + 2]
  double* loc = data + slice + 2;                                      // [cpc][4] chunk moments
  double* gat = loc + 4 * cpc;                                         // [2][gsz][4] (as leader)
  Shared* sh = reinterpret_cast<Shared*>(gat + 8 * gsz);

  const int cluster_id = blockIdx.x / cs;
  const int n_clusters = gridDim.x / cs;
  const int words_cta = slice / 32;
  const int lo = (int)rank * slice;

  if (tid == 0) {
    for (int j = 0; j < kMaxStages; ++j) mbar_init(&sh->bar[j], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sh->gat_bar[b], 1);
      mbar_init(&sh->res_bar[b], 1);
    }
    fence_mbar_init();
  }
  cluster_sync();      // barriers initialised cluster-wide before any remote signal

  if (c.exhaustive) {
    // thresholds and means are -inf (engine.py:29-32): every valid slot is in
    // C0 and passes the filter; no table bytes are needed.
    for (int item = cluster_id; item < n_items; item += n_clusters) {
      if (c.bypass[item >> 1]) continue;
      const Item it = make_item(c, item, n_items, slice, lo);
      uint32_t* b0 = c.bits + ((size_t)item * 2 + 0) * c.words;
      uint32_t* bf = c.bits + ((size_t)item * 2 + 1) * c.words;
      for (int w = tid; w < words_cta; w += kThreads) {
        const int valid = max(0, min(32, it.cnt - w * 32));
        const uint32_t word = valid == 32 ? LFPS_FULL : ((1u << valid) - 1u);
        b0[lo / 32 + w] = word;
        bf[lo / 32 + w] = word;
      }
      if (rank == 0 && tid == 0) {
        double* thr = c.thr + (size_t)item * 4;
        thr[0] = -INFINITY; thr[1] = -INFINITY; thr[2] = 0.0; thr[3] = NAN;
      }
    }
    cluster_sync();
    return;
  }

  int trace_it = 0;
  unsigned long long* trace = reinterpret_cast<unsigned long long*>(c.scratch);
#define TS(k)                                                                        \
  do {                                                                               \
    if constexpr (MODE == 3) {                                                       \
      if (cluster_id == 0 && tid == 0 && trace_it < 16)                              \
        trace[((size_t)rank * 16 + trace_it) * 12 + (k)] = gtimer();                 \
    }                                                                                \
  } while (0)

  // software pipeline over this cluster's non-bypassed items: the copy of
  // item k+1 is in flight while item k's thresholds are merged and the bits
  // of item k-1 are written
  int item = next_valid(c, cluster_id, n_items, n_clusters);
  Item cur = make_item(c, item, n_items, slice, lo);
  int item_n = next_valid(c, item + n_clusters, n_items, n_clusters);
  Item nxt = make_item(c, item_n, n_items, slice, lo);
  if (warp == 0 && item < n_items) {
    issue_copies(c, cur, data, sh, lo, lane);
    if (lane == 16 && item_n < n_items) prefetch_slice(c, nxt, lo);
    if (lane == 17) mbar_expect_tx(&sh->res_bar[0], 24u);
    if (lane == 18 && rank == 0) mbar_expect_tx(&sh->gat_bar[0], (uint32_t)gsz * 32u);
  }
  Item prev;
  prev.item = n_items;
  uint32_t pc = 0;                 // processed items (uniform across the cluster)
  uint32_t gph[2] = {0u, 0u};      // this CTA's completed gather phases per buffer

  while (item < n_items) {
    TS(0);
    const uint32_t b = pc & 1u;
    const int leader = (int)(pc % (uint32_t)cs);
    const uint32_t gat_l = map_rank(smem_u32(gat + 4 * b * gsz), leader);
    const uint32_t gbar_l = map_rank(smem_u32(&sh->gat_bar[b]), leader);

    // ---- (1) chunk moments of the resident slice ------------------------------
    for (int ch = warp; ch < cpc; ch += kWarps) {
      const int i0 = ch * kChunk;
      const int vc = max(0, min(kChunk, cur.cnt - i0));
      double mu = 0.0, m2 = 0.0, m3 = 0.0, m4 = 0.0;
      if (vc > 0) {
        mbar_wait(&sh->bar[(cur.off + i0) / kStage], pc & 1u);
        mbar_wait(&sh->bar[(cur.off + i0 + vc - 1) / kStage], pc & 1u);
        const double* src = data + cur.off + i0 + lane;
        double v[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = (e * 32 + lane < vc) ? src[e * 32] : 0.0;
        double q[4];
#pragma unroll
        for (int gq = 0; gq < 4; ++gq)
          q[gq] = cadd(cadd(v[4 * gq], v[4 * gq + 1]), cadd(v[4 * gq + 2], v[4 * gq + 3]));
        mu = cdiv_count(warp_fold(cadd(cadd(q[0], q[1]), cadd(q[2], q[3]))), (double)vc);
        double p2[4], p3[4], p4[4];
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) {
          double t2[4], t3[4], t4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int e = 4 * gq + t;
            const double d = (e * 32 + lane < vc) ? csub(v[e], mu) : 0.0;
            const double d2 = cmul(d, d);
            t2[t] = d2;
            t3[t] = cmul(d2, d);
            t4[t] = cmul(d2, d2);
          }
          p2[gq] = cadd(cadd(t2[0], t2[1]), cadd(t2[2], t2[3]));
          p3[gq] = cadd(cadd(t3[0], t3[1]), cadd(t3[2], t3[3]));
          p4[gq] = cadd(cadd(t4[0], t4[1]), cadd(t4[2], t4[3]));
        }
        m2 = warp_fold(cadd(cadd(p2[0], p2[1]), cadd(p2[2], p2[3])));
        m3 = warp_fold(cadd(cadd(p3[0], p3[1]), cadd(p3[2], p3[3])));
        m4 = warp_fold(cadd(cadd(p4[0], p4[1]), cadd(p4[2], p4[3])));
      }
      if (lane == 0) {
        loc[4 * ch] = mu;
        loc[4 * ch + 1] = m2;
        loc[4 * ch + 2] = m3;
        loc[4 * ch + 3] = m4;
      }
    }
    __syncthreads();                  // smem slice consumed
    TS(1);
    // ---- (2) aligned 8-chunk group merges -> leader; next item's copy -------------
    if (warp < gpc) {
      const int ch = warp * kGroup + (lane & 7);
      Mom a;
      a.n = (double)max(0, min(kChunk, cur.cnt - ch * kChunk));
      a.mu = loc[4 * ch];
      a.m2 = loc[4 * ch + 1];
      a.m3 = loc[4 * ch + 2];
      a.m4 = loc[4 * ch + 3];
#pragma unroll
      for (int h = 1; h < kGroup; h <<= 1) {
        const Mom o = shfl_mom(a, h);
        a = (lane & h) ? merge(o, a) : merge(a, o);
      }
      if (lane == 0) {
        const uint32_t dst = gat_l + (uint32_t)(rank * gpc + warp) * 32u;
        st_async_v2f64(dst, a.mu, a.m2, gbar_l);
        st_async_v2f64(dst + 16u, a.m3, a.m4, gbar_l);
      }
    } else if (warp == gpc) {
      if (item_n < n_items) issue_copies(c, nxt, data, sh, lo, lane);
    }
    // look one more item ahead: metadata + L2 prefetch
    const int item_nn = next_valid(c, item_n + n_clusters, n_items, n_clusters);
    const Item nn = make_item(c, item_nn, n_items, slice, lo);
    if (warp == gpc && lane == 31 && item_nn < n_items) prefetch_slice(c, nn, lo);
    TS(2);

    // ---- (3) leader: merge -> thresholds -> broadcast ---------------------------
    if ((int)rank == leader && warp == 0) {
      mbar_wait(&sh->gat_bar[b], gph[b] & 1u);
      gph[b] += 1;
      TS(8);
      const Mom tot = merge_tree(gat + 4 * b * gsz, (cur.m + kGroupSlots - 1) / kGroupSlots,
                                 cur.m, lane);
      double thr0 = NAN, thrf = 0.0, degf = 0.0;
      if (lane == 0) {
        const double mean = cmul(tot.mu, cur.sc);
        const bool deg = cmul(cmul(tot.m2, cur.sc), cur.sc) < 1e-12;
        double tau = NAN, kappa = NAN;
        if (!deg) {
          kappa = cdiv(tot.m4, cmul(tot.m2, tot.m2));
          if (kappa == 0.0) set_err(c, cur.s, LFPS_ERR_KAPPA_ZERO);
          tau = cdiv(cmul(c.a, mean), kappa);
          thr0 = cdiv(tau, cur.sc);
        }
        thrf = cdiv(mean, cur.sc);
        degf = deg ? 1.0 : 0.0;
        double* thr = c.thr + (size_t)cur.item * 4;
        thr[0] = tau; thr[1] = mean; thr[2] = degf; thr[3] = kappa;
      }
      thr0 = __shfl_sync(LFPS_FULL, thr0, 0);
      thrf = __shfl_sync(LFPS_FULL, thrf, 0);
      degf = __shfl_sync(LFPS_FULL, degf, 0);
      if (lane < cs) {
        const uint32_t dst = map_rank(smem_u32(&sh->bcast[b][0]), lane);
        const uint32_t bar = map_rank(smem_u32(&sh->res_bar[b]), lane);
        st_async_v2f64(dst, thr0, thrf, bar);
        st_async_f64(dst + 16u, degf, bar);
      }
    }
    TS(3);

    // ---- (4) bits of the previous item (its thresholds are in) ------------------
    if (prev.item < n_items) {
      const uint32_t pb = (pc - 1) & 1u;
      mbar_wait(&sh->res_bar[pb], ((pc - 1) >> 1) & 1u);
      const bool deg = sh->bcast[pb][2] != 0.0;
      const long long tb0 = deg ? 0x7fffffffffffffffll : thr_bits(sh->bcast[pb][0]);
      const long long tbf = thr_bits(sh->bcast[pb][1]);
      slice_bits(c, prev, lo, words_cta, tb0, tbf, warp, lane);
      __syncthreads();                // bcast[pb] read by everyone before re-arming
    }
    // arm the barriers of item pc + 1 (their previous phases are complete)
    if (tid == 0 && item_n < n_items) {
      mbar_expect_tx(&sh->res_bar[(pc + 1) & 1u], 24u);
      if ((int)rank == (int)((pc + 1) % (uint32_t)cs))
        mbar_expect_tx(&sh->gat_bar[(pc + 1) & 1u], (uint32_t)gsz * 32u);
    }
    TS(6);
    prev = cur;
    cur = nxt;
    nxt = nn;
    item = item_n;
    item_n = item_nn;
    ++pc;
    ++trace_it;
  }
  // bits of the last item
  if (prev.item < n_items) {
    const uint32_t pb = (pc - 1) & 1u;
    mbar_wait(&sh->res_bar[pb], ((pc - 1) >> 1) & 1u);
    const bool deg = sh->bcast[pb][2] != 0.0;
    const long long tb0 = deg ? 0x7fffffffffffffffll : thr_bits(sh->bcast[pb][0]);
    const long long tbf = thr_bits(sh->bcast[pb][1]);
    slice_bits(c, prev, lo, words_cta, tb0, tbf, warp, lane);
  }
  cluster_sync();        // no CTA leaves while a peer may still address it
#undef TS
}

struct ScanLaunch {
  int slice = 0, cs = 0, clusters = 0;
  size_t smem = 0;
};

}  // namespace

template <int MODE>
cudaError_t launch_scan_t(const Ctx& c, int m_max, cudaStream_t st, int slice_override) {
  // slice: multiple of 4096 so CTAs own whole aligned 8-chunk groups; <= 16 CTAs
  int slice = ((m_max + 15) / 16 + kGroupSlots - 1) / kGroupSlots * kGroupSlots;
  if (slice < kGroupSlots) slice = kGroupSlots;
  if (slice_override > 0) slice = slice_override;
  if (slice > kMaxSlice || slice % kGroupSlots) return cudaErrorInvalidValue;
  int cs = (m_max + slice - 1) / slice;
  if (cs < 1) cs = 1;
  if (cs > 16) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(slice + 2) * 8 + 4 * (size_t)(slice / kChunk) * 8 +
                      8 * (size_t)cs * (slice / kGroupSlots) * 8 + sizeof(Shared);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static ScanLaunch cache;
  if (cache.slice != slice || cache.cs != cs || cache.smem != smem) {
    cudaFuncSetAttribute(scan_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(scan_kernel<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cfg.gridDim = dim3(cs * 64, 1, 1);
    int clusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, scan_kernel<MODE>, &cfg);
    if (e != cudaSuccess || clusters < 1) clusters = 148 / cs;
    if (clusters < 1) clusters = 1;
    cache = {slice, cs, clusters, smem};
  }
  const int n_items = 2 * c.NS;
  int clusters = cache.clusters;
  if (clusters > n_items) clusters = n_items;
  cfg.gridDim = dim3(cs * clusters, 1, 1);
  return cudaLaunchKernelEx(&cfg, scan_kernel<MODE>, c, slice, n_items);
}

cudaError_t launch_scan(const Ctx& c, int m_max, cudaStream_t st) {
  return launch_scan_t<0>(c, m_max, st, 0);
}

cudaError_t launch_scan_experiment(const Ctx& c, int m_max, int mode, int slice, cudaStream_t st) {
  switch (mode) {
    case 0: return launch_scan_t<0>(c, m_max, st, slice);
    case 3: return launch_scan_t<3>(c, m_max, st, slice);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
