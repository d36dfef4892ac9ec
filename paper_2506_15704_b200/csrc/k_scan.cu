// k_scan.cu -- tracker-table scan (K1 moments + the threshold half of K2).
//
// Persistent thread-block clusters; cluster c walks the (session, table)
// items c, c + NC, c + 2 NC, ...  Each CTA of a cluster owns a contiguous
// slice of the item's logical range and keeps it in shared memory for the
// whole item, so the table is read from HBM exactly once:
//
//   load    1-D bulk async copies (cp.async.bulk + mbarrier) of the slice,
//           served from L2: while item i is processed, the slice of item
//           i + NC was already requested with cp.async.bulk.prefetch.L2, so
//           HBM streams continuously underneath the compute phases
//   pass 1  chunk sums            -> cluster-wide mean   (DSMEM gather)
//   pass 2  centred c^2, c^4 sums -> cluster-wide s2, s4  (DSMEM gather)
//           thresholds tau / mean / degenerate (tables.py:295-317)
//   pass 3  ballot bitmaps: C0 bit = phys > tau/scale (select_initial,
//           candidates.py:45-58), F bit = phys > mean/scale (the expansion
//           filter, candidates.py:79-81) -> workspace (1/32 of the bytes)
//
// Summation order is canonical (devmath.table_sum): 512-element warp
// chunks, lane-strided, folded, then a pairwise tree over all chunk partials
// of the table -- independent of the cluster shape.
#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 512;          // canonical chunk (devmath.TABLE_CHUNK)
constexpr int kStage = 1024;         // elements per bulk-copy stage (8 KB)
constexpr int kMaxStages = 12;
constexpr int kMaxSlice = kStage * kMaxStages - 2;  // smem elements incl. slack
constexpr int kTreeLeaves = 512;     // >= chunks of the largest supported table
constexpr int kLeavesPerLane = kTreeLeaves / 32;

struct Shared {
  uint64_t bar[kMaxStages];   // bulk-copy stages
  uint64_t gat_bar;           // leader: partials of the cluster have landed
  uint64_t res_bar;           // every CTA: the leader's reduction result landed
  double bcast[2];            // reduction results (mean_p) / (s2_p, s4_p)
};

// Canonical pairwise tree over the leader's gathered chunk partials
// (kTreeLeaves zero-padded leaves; lane l owns leaves [16 l, 16 l + 16)).
template <int STRIDE>
__device__ __forceinline__ double leader_tree(const double* g, int n_chunks, int lane) {
  double v[kLeavesPerLane];
#pragma unroll
  for (int k = 0; k < kLeavesPerLane; ++k) {
    const int i = lane * kLeavesPerLane + k;
    v[k] = i < n_chunks ? g[i * STRIDE] : 0.0;
  }
#pragma unroll
  for (int h = 1; h < kLeavesPerLane; h <<= 1) {
#pragma unroll
    for (int k = 0; k < kLeavesPerLane; k += 2 * h) v[k] = cadd(v[k], v[k + h]);
  }
  double acc = v[0];
#pragma unroll
  for (int h = 1; h <= 16; h <<= 1) acc = cadd(acc, __shfl_xor_sync(LFPS_FULL, acc, h));
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

// MODE (experiments only, tools/scan_bench.cu): 0 = full kernel, 1 = load
// only, 2 = load + pass 1 + first cluster reduction, 3 = full kernel with a
// per-phase globaltimer trace of cluster 0 written to c.scratch.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 3) scan_kernel(Ctx c, int slice, int n_items) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cs = (int)cluster_size();
  const int cpc = slice / kChunk;                // chunks per CTA
  double* data = reinterpret_cast<double*>(smem_raw);                 // [slice + 2]
  double* g1 = data + slice + 2;                                       // [cs * cpc] leader
  double* g2 = g1 + cs * cpc;                                          // [cs * cpc][2] leader
  Shared* sh = reinterpret_cast<Shared*>(g2 + 2 * cs * cpc);

  const int cluster_id = blockIdx.x / cs;
  const int n_clusters = gridDim.x / cs;
  const int words_cta = slice / 32;
  const int lo = (int)rank * slice;
  // shared::cluster addresses of the leader's gather buffers / barrier and
  // of every CTA's result slot / barrier (rank-symmetric layout)
  const uint32_t g1_lead = map_rank(smem_u32(g1), 0);
  const uint32_t g2_lead = map_rank(smem_u32(g2), 0);
  const uint32_t gat_lead = map_rank(smem_u32(&sh->gat_bar), 0);

  if (tid == 0) {
    for (int j = 0; j < kMaxStages; ++j) mbar_init(&sh->bar[j], 1);
    mbar_init(&sh->gat_bar, 1);
    mbar_init(&sh->res_bar, 1);
    fence_mbar_init();
  }
  Meta cur = load_meta(c, cluster_id, n_items);
  Meta nxt = load_meta(c, cluster_id + n_clusters, n_items);
  if (tid == 0) prefetch_item(c, cluster_id, cur, slice, rank);
  cluster_sync();      // barriers initialised cluster-wide before any remote signal
  uint32_t ph = 0;     // completed phases per stage barrier (one per item)
  int trace_it = 0;
  unsigned long long* trace = reinterpret_cast<unsigned long long*>(c.scratch);
#define TS(k)                                                                        \
  do {                                                                               \
    if constexpr (MODE == 3) {                                                       \
      if (cluster_id == 0 && tid == 0 && trace_it < 16)                              \
        trace[((size_t)rank * 16 + trace_it) * 12 + (k)] = gtimer();                 \
    }                                                                                \
  } while (0)

  for (int item = cluster_id; item < n_items; item += n_clusters) {
    const int s = item >> 1, table = item & 1;
    const Meta mt = cur;
    cur = nxt;
    nxt = load_meta(c, item + 2 * n_clusters, n_items);   // in flight during this item
    if (mt.byp) continue;                        // uniform across the cluster
    const int m = mt.m;
    const int cnt = max(0, min(slice, m - lo));
    uint32_t* bits_c0 = c.bits + ((size_t)(s * 2 + table) * 2 + 0) * c.words;
    uint32_t* bits_f = c.bits + ((size_t)(s * 2 + table) * 2 + 1) * c.words;

    if (c.exhaustive) {
      // thresholds and means are -inf (engine.py:29-32): every valid slot is
      // in C0 and passes the filter; no table bytes are needed.
      for (int w = tid; w < words_cta; w += kThreads) {
        const int valid = max(0, min(32, cnt - w * 32));
        const uint32_t word = valid == 32 ? LFPS_FULL : ((1u << valid) - 1u);
        bits_c0[lo / 32 + w] = word;
        bits_f[lo / 32 + w] = word;
      }
      if (rank == 0 && tid == 0) {
        double* thr = c.thr + (size_t)(s * 2 + table) * 4;
        thr[0] = -INFINITY; thr[1] = -INFINITY; thr[2] = 0.0; thr[3] = NAN;
      }
      continue;
    }

    TS(0);
    // ---- stage the slice into shared memory (L2 hits after the prefetch) ----
    const int off = slice_off(c, table, mt.base, lo);
    const int total = cnt > 0 ? ((off + cnt + 1) & ~1) : 0;   // even element count
    const int nst = (total + kStage - 1) / kStage;
    if (tid == 0) {
      fence_proxy_async();   // generic reads of the previous item before async writes
      for (int j = 0; j < kMaxStages; ++j) {
        if (j < nst) {
          const int e0 = j * kStage;
          const int len = min(kStage, total - e0);
          mbar_expect_tx(&sh->bar[j], (uint32_t)len * 8u);
          Piece pc[2];
          const int np = table_pieces(c, s, table, mt.base, lo - off + e0, len, pc);
          int at = e0;
          for (int k = 0; k < np; ++k) {
            bulk_g2s(data + at, pc[k].p, (uint32_t)pc[k].n * 8u, &sh->bar[j]);
            at += pc[k].n;
          }
        } else {
          mbar_arrive(&sh->bar[j]);            // keep every stage's phase in step
        }
      }
      // arm the reduction barriers for this item's first reduction
      if constexpr (MODE != 1) {
        mbar_expect_tx(&sh->res_bar, 8u);
        if (rank == 0) mbar_expect_tx(&sh->gat_bar, (uint32_t)(cs * cpc) * 8u);
      }
      if (item + n_clusters < n_items) prefetch_item(c, item + n_clusters, cur, slice, rank);
    }
    TS(1);
    const uint32_t par = ph & 1u;
    ++ph;
    if constexpr (MODE == 1) {
      if (cnt > 0) {
        for (int j = warp; j < nst; j += kWarps) mbar_wait(&sh->bar[j], par);
      }
      __syncthreads();
      continue;
    }

    // ---- pass 1: chunk sums, each sent straight to the leader ----------------
    for (int ch = warp; ch < cpc; ch += kWarps) {
      const int i0 = ch * kChunk;
      const int vc = max(0, min(kChunk, cnt - i0));
      double acc = 0.0;
      if (vc > 0) {
        mbar_wait(&sh->bar[(off + i0) / kStage], par);
        mbar_wait(&sh->bar[(off + i0 + vc - 1) / kStage], par);
        const double* src = data + off + i0 + lane;
        // adjacent-pair tree over the lane's 16 elements, built 4 at a time
        double q4[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          double v[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int e = 4 * g + t;
            v[t] = (vc == kChunk || i0 + e * 32 + lane < cnt) ? src[e * 32] : 0.0;
          }
          q4[g] = cadd(cadd(v[0], v[1]), cadd(v[2], v[3]));
        }
        acc = warp_fold(cadd(cadd(q4[0], q4[1]), cadd(q4[2], q4[3])));
      }
      if (lane == 0) st_async_f64(g1_lead + (uint32_t)(rank * cpc + ch) * 8u, acc, gat_lead);
    }
    const int n_chunks = (m + kChunk - 1) / kChunk;
    TS(2);
    if (rank == 0 && warp == 0) {
      mbar_wait(&sh->gat_bar, 0);
      TS(8);
      const double mean_p = cdiv(leader_tree<1>(g1, n_chunks, lane), (double)m);
      if (lane == 0) {                            // arm reduction 2
        if constexpr (MODE == 2) mbar_arrive(&sh->gat_bar);
        else mbar_expect_tx(&sh->gat_bar, (uint32_t)(cs * cpc) * 16u);
      }
      if (lane < cs) {
        st_async_f64(map_rank(smem_u32(&sh->bcast[0]), lane), mean_p,
                     map_rank(smem_u32(&sh->res_bar), lane));
      }
    }
    mbar_wait(&sh->res_bar, 0);
    TS(3);
    const double mean_p = sh->bcast[0];
    __syncthreads();                              // everyone read bcast before re-arming
    if constexpr (MODE == 2) {
      // close reduction 2 with no payload so the barrier phases stay aligned
      if (tid == 0) mbar_arrive(&sh->res_bar);
      if (rank == 0 && tid == 0) c.thr[(size_t)(s * 2 + table) * 4] = mean_p;
      mbar_wait(&sh->res_bar, 1);
      __syncthreads();
      continue;
    }
    if (tid == 0) mbar_expect_tx(&sh->res_bar, 16u);

    // ---- pass 2: centred second and fourth powers -----------------------------
    for (int ch = warp; ch < cpc; ch += kWarps) {
      const int i0 = ch * kChunk;
      double a2 = 0.0, a4 = 0.0;
      if (i0 < cnt) {
        const double* src = data + off + i0 + lane;
        const bool full = i0 + kChunk <= cnt;
        double p2[4], p4[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          double v2[4], v4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int e = 4 * g + t;
            const bool ok = full || i0 + e * 32 + lane < cnt;
            const double x = csub(ok ? src[e * 32] : mean_p, mean_p);
            const double x2 = cmul(x, x);
            v2[t] = ok ? x2 : 0.0;
            v4[t] = ok ? cmul(x2, x2) : 0.0;
          }
          p2[g] = cadd(cadd(v2[0], v2[1]), cadd(v2[2], v2[3]));
          p4[g] = cadd(cadd(v4[0], v4[1]), cadd(v4[2], v4[3]));
        }
        a2 = warp_fold(cadd(cadd(p2[0], p2[1]), cadd(p2[2], p2[3])));
        a4 = warp_fold(cadd(cadd(p4[0], p4[1]), cadd(p4[2], p4[3])));
      }
      if (lane == 0) st_async_v2f64(g2_lead + (uint32_t)(rank * cpc + ch) * 16u, a2, a4, gat_lead);
    }
    TS(4);
    if (rank == 0 && warp == 0) {
      mbar_wait(&sh->gat_bar, 1);
      TS(9);
      const double t2 = leader_tree<2>(g2, n_chunks, lane);
      const double t4 = leader_tree<2>(g2 + 1, n_chunks, lane);
      if (lane < cs) {
        st_async_v2f64(map_rank(smem_u32(&sh->bcast[0]), lane), t2, t4,
                       map_rank(smem_u32(&sh->res_bar), lane));
      }
    }
    mbar_wait(&sh->res_bar, 1);
    TS(5);

    // ---- thresholds (tables.py:305-317, candidates.py:52-54), every CTA ------
    const double sc = mt.sc;
    const double s2p = sh->bcast[0], s4p = sh->bcast[1];
    const double mean = cmul(mean_p, sc);
    const bool deg = cmul(cmul(s2p, sc), sc) < 1e-12;
    double tau = NAN, kappa = NAN, thr0 = NAN;
    if (!deg) {
      kappa = cdiv(s4p, cmul(s2p, s2p));
      tau = cdiv(cmul(c.a, mean), kappa);
      thr0 = cdiv(tau, sc);
    }
    const double thrf = cdiv(mean, sc);
    if (rank == 0 && tid == 0) {
      if (!deg && kappa == 0.0) set_err(c, s, LFPS_ERR_KAPPA_ZERO);
      double* thr = c.thr + (size_t)(s * 2 + table) * 4;
      thr[0] = tau; thr[1] = mean; thr[2] = deg ? 1.0 : 0.0; thr[3] = kappa;
    }

    // ---- pass 3: ballot bitmaps ------------------------------------------------
    const long long tb0 = deg ? 0x7fffffffffffffffll : thr_bits(thr0);
    const long long tbf = thr_bits(thrf);
    for (int g0 = warp * 32; g0 < words_cta; g0 += kWarps * 32) {
      uint32_t my0 = 0, myf = 0;
      const int nw = min(32, words_cta - g0);
      const long long* src = reinterpret_cast<const long long*>(data + off) + g0 * 32 + lane;
      if (nw == 32 && (g0 + 32) * 32 <= cnt) {
        // full group: batched loads, integer compares, no masking
#pragma unroll
        for (int jb = 0; jb < 32; jb += 8) {
          long long x[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) x[t] = src[(jb + t) * 32];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const uint32_t w0 = __ballot_sync(LFPS_FULL, x[t] > tb0);
            const uint32_t wf = __ballot_sync(LFPS_FULL, x[t] > tbf);
            if (lane == jb + t) { my0 = w0; myf = wf; }
          }
        }
      } else {
        for (int j = 0; j < nw; ++j) {
          const bool valid = (g0 + j) * 32 + lane < cnt;
          const long long x = valid ? src[j * 32] : 0ll;
          const uint32_t w0 = __ballot_sync(LFPS_FULL, valid && x > tb0);
          const uint32_t wf = __ballot_sync(LFPS_FULL, valid && x > tbf);
          if (lane == j) { my0 = w0; myf = wf; }
        }
      }
      if (lane < nw) {
        bits_c0[lo / 32 + g0 + lane] = my0;
        bits_f[lo / 32 + g0 + lane] = myf;
      }
    }
    TS(6);
    __syncthreads();     // slice and bcast are free for the next item
    TS(7);
    ++trace_it;
  }
  cluster_sync();        // no CTA leaves while a peer may still address it
}

struct ScanLaunch {
  int slice = 0, cs = 0, clusters = 0;
  size_t smem = 0;
};

}  // namespace

template <int MODE>
cudaError_t launch_scan_t(const Ctx& c, int m_max, cudaStream_t st, int slice_override) {
  // slice: multiple of 512 so CTAs own whole canonical chunks; <= 16 CTAs
  int slice = ((m_max + 15) / 16 + kChunk - 1) / kChunk * kChunk;
  if (slice < 1024) slice = 1024;
  if (slice_override > 0) slice = slice_override;
  if (slice > kMaxSlice / kChunk * kChunk) return cudaErrorInvalidValue;
  int cs = (m_max + slice - 1) / slice;
  if (cs < 1) cs = 1;
  if (cs > 16) return cudaErrorInvalidValue;
  const size_t smem = (size_t)(slice + 2) * 8 + 3 * (size_t)cs * (slice / kChunk) * 8 + sizeof(Shared);
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
    case 1: return launch_scan_t<1>(c, m_max, st, slice);
    case 2: return launch_scan_t<2>(c, m_max, st, slice);
    case 3: return launch_scan_t<3>(c, m_max, st, slice);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
