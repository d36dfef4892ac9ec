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
  uint64_t bar[kMaxStages];
  double bcast[8];
};

// Canonical sum of all chunk partials of the cluster (pairwise tree over
// kTreeLeaves zero-padded leaves; lane l owns leaves [16 l, 16 l + 16)).
__device__ __forceinline__ double cluster_tree(uint32_t part_saddr, int chunks_per_cta,
                                               int n_chunks, int lane) {
  double v[kLeavesPerLane];
#pragma unroll
  for (int k = 0; k < kLeavesPerLane; ++k) {
    const int i = lane * kLeavesPerLane + k;
    v[k] = 0.0;
    if (i < n_chunks) {
      const uint32_t owner = i / chunks_per_cta;
      const uint32_t li = i - owner * chunks_per_cta;
      v[k] = ld_cluster_f64(map_rank(part_saddr + li * 8u, owner));
    }
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

// Byte range [ptr, ptr + bytes) pieces of logical range [l0, l0 + len) of a
// table (ver: contiguous; sla: ring of C slots).  Returns piece count (1-2).
struct Piece {
  const double* p;
  int n;
};
__device__ __forceinline__ int table_pieces(const Ctx& c, int s, int table, int l0, int len,
                                            Piece* out) {
  if (table == 0) {
    out[0] = {c.ver + (size_t)s * c.m_cap + l0, len};
    return 1;
  }
  const int C = c.ring_cap;
  const double* ring = c.sla + (size_t)s * C;
  const int p = ((c.sla_base[s] + l0) % C + C) % C;
  const int first = min(len, C - p);
  out[0] = {ring + p, first};
  if (first < len) {
    out[1] = {ring, len - first};
    return 2;
  }
  return 1;
}

// smem element e <-> logical (lo - off + e); off keeps copies 16-B aligned
__device__ __forceinline__ int slice_off(const Ctx& c, int s, int table, int lo) {
  return table == 1 ? (((c.sla_base[s] + lo) % c.ring_cap) & 1) : 0;
}

__device__ __forceinline__ void prefetch_item(const Ctx& c, int item, int n_items, int slice,
                                              uint32_t rank) {
  if (item >= n_items) return;
  const int s = item >> 1, table = item & 1;
  if (c.exhaustive || c.bypass[s]) return;
  const int m = c.n_ctx[s / c.Hq] - c.S;
  const int lo = (int)rank * slice;
  const int cnt = max(0, min(slice, m - lo));
  if (cnt == 0) return;
  const int off = slice_off(c, s, table, lo);
  const int total = (off + cnt + 1) & ~1;
  Piece pc[2];
  const int np = table_pieces(c, s, table, lo - off, total, pc);
  for (int k = 0; k < np; ++k) prefetch_l2(pc[k].p, (uint32_t)pc[k].n * 8u);
}

__global__ void __launch_bounds__(kThreads) scan_kernel(Ctx c, int slice, int n_items) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* data = reinterpret_cast<double*>(smem_raw);                 // [slice + 2]
  double* part1 = data + slice + 2;                                    // [slice / 512]
  double* part2 = part1 + slice / kChunk;
  double* part4 = part2 + slice / kChunk;
  Shared* sh = reinterpret_cast<Shared*>(part4 + slice / kChunk);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cs = (int)cluster_size();
  const int cluster_id = blockIdx.x / cs;
  const int n_clusters = gridDim.x / cs;
  const int cpc = slice / kChunk;                // chunks per CTA
  const int words_cta = slice / 32;
  const int lo = (int)rank * slice;

  if (tid == 0) {
    for (int j = 0; j < kMaxStages; ++j) mbar_init(&sh->bar[j], 1);
    fence_mbar_init();
    prefetch_item(c, cluster_id, n_items, slice, rank);
  }
  __syncthreads();
  uint32_t ph = 0;   // completed phases per stage barrier

  for (int item = cluster_id; item < n_items; item += n_clusters) {
    const int s = item >> 1, table = item & 1;
    if (c.bypass[s]) continue;                   // uniform across the cluster
    const int m = c.n_ctx[s / c.Hq] - c.S;
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

    // ---- stage the slice into shared memory (L2 hits after the prefetch) --
    const int off = slice_off(c, s, table, lo);
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
          const int np = table_pieces(c, s, table, lo - off + e0, len, pc);
          int at = e0;
          for (int k = 0; k < np; ++k) {
            bulk_g2s(data + at, pc[k].p, (uint32_t)pc[k].n * 8u, &sh->bar[j]);
            at += pc[k].n;
          }
        } else {
          mbar_arrive(&sh->bar[j]);            // keep every stage's phase in step
        }
      }
      prefetch_item(c, item + n_clusters, n_items, slice, rank);
    }
    const uint32_t par = ph & 1u;
    ++ph;

    // ---- pass 1: chunk sums ---------------------------------------------------
    for (int ch = warp; ch < cpc; ch += kWarps) {
      const int i0 = ch * kChunk;
      const int vc = max(0, min(kChunk, cnt - i0));
      double acc = 0.0;
      if (vc > 0) {
        mbar_wait(&sh->bar[(off + i0) / kStage], par);
        mbar_wait(&sh->bar[(off + i0 + vc - 1) / kStage], par);
        const double* src = data + off + i0 + lane;
        if (vc == kChunk) {
#pragma unroll
          for (int e = 0; e < kChunk / 32; ++e) acc = cadd(acc, src[e * 32]);
        } else {
          for (int e = 0; e < kChunk / 32; ++e)
            if (i0 + e * 32 + lane < cnt) acc = cadd(acc, src[e * 32]);
        }
        acc = warp_fold(acc);
      }
      if (lane == 0) part1[ch] = acc;
    }
    cluster_sync();
    const int n_chunks = (m + kChunk - 1) / kChunk;
    if (warp == 0) {
      const double tot = cluster_tree(smem_u32(part1), cpc, n_chunks, lane);
      if (lane == 0) sh->bcast[0] = cdiv(tot, (double)m);
    }
    __syncthreads();
    const double mean_p = sh->bcast[0];

    // ---- pass 2: centred second and fourth powers -----------------------------
    for (int ch = warp; ch < cpc; ch += kWarps) {
      const int i0 = ch * kChunk;
      double a2 = 0.0, a4 = 0.0;
      if (i0 < cnt) {
        const double* src = data + off + i0 + lane;
        if (i0 + kChunk <= cnt) {
#pragma unroll
          for (int e = 0; e < kChunk / 32; ++e) {
            const double x = csub(src[e * 32], mean_p);
            const double x2 = cmul(x, x);
            a2 = cadd(a2, x2);
            a4 = cadd(a4, cmul(x2, x2));
          }
        } else {
          for (int e = 0; e < kChunk / 32; ++e) {
            if (i0 + e * 32 + lane < cnt) {
              const double x = csub(src[e * 32], mean_p);
              const double x2 = cmul(x, x);
              a2 = cadd(a2, x2);
              a4 = cadd(a4, cmul(x2, x2));
            }
          }
        }
        a2 = warp_fold(a2);
        a4 = warp_fold(a4);
      }
      if (lane == 0) { part2[ch] = a2; part4[ch] = a4; }
    }
    cluster_sync();
    if (warp == 0) {
      const double t2 = cluster_tree(smem_u32(part2), cpc, n_chunks, lane);
      if (lane == 0) sh->bcast[1] = t2;
    } else if (warp == 1) {
      const double t4 = cluster_tree(smem_u32(part4), cpc, n_chunks, lane);
      if (lane == 0) sh->bcast[2] = t4;
    }
    __syncthreads();

    // ---- thresholds (tables.py:305-317, candidates.py:52-54) ----------------
    if (tid == 0) {
      const double sc = c.scale[s];
      const double s2p = sh->bcast[1], s4p = sh->bcast[2];
      const double mean = cmul(mean_p, sc);
      const double s2 = cmul(cmul(s2p, sc), sc);
      const bool deg = s2 < 1e-12;
      double tau = NAN, kappa = NAN, thr0 = NAN;
      if (!deg) {
        kappa = cdiv(s4p, cmul(s2p, s2p));
        if (kappa == 0.0 && rank == 0) set_err(c, s, LFPS_ERR_KAPPA_ZERO);
        tau = cdiv(cmul(c.a, mean), kappa);
        thr0 = cdiv(tau, sc);
      }
      sh->bcast[3] = thr0;
      sh->bcast[4] = cdiv(mean, sc);
      sh->bcast[5] = deg ? 1.0 : 0.0;
      if (rank == 0) {
        double* thr = c.thr + (size_t)(s * 2 + table) * 4;
        thr[0] = tau; thr[1] = mean; thr[2] = deg ? 1.0 : 0.0; thr[3] = kappa;
      }
    }
    __syncthreads();
    const double thr0 = sh->bcast[3], thrf = sh->bcast[4];
    const bool deg = sh->bcast[5] != 0.0;

    // ---- pass 3: ballot bitmaps ------------------------------------------------
    for (int g0 = warp * 32; g0 < words_cta; g0 += kWarps * 32) {
      uint32_t my0 = 0, myf = 0;
      const int nw = min(32, words_cta - g0);
      for (int j = 0; j < nw; ++j) {
        const int i = (g0 + j) * 32 + lane;
        const bool valid = i < cnt;
        const double x = valid ? data[off + i] : 0.0;
        const uint32_t w0 = __ballot_sync(LFPS_FULL, valid && !deg && x > thr0);
        const uint32_t wf = __ballot_sync(LFPS_FULL, valid && x > thrf);
        if (lane == j) { my0 = w0; myf = wf; }
      }
      if (lane < nw) {
        bits_c0[lo / 32 + g0 + lane] = my0;
        bits_f[lo / 32 + g0 + lane] = myf;
      }
    }
    __syncthreads();     // the smem slice is free for the next item's copies
  }
  // peers may still read this CTA's partials of the last item
  cluster_sync();
}

struct ScanLaunch {
  int slice = 0, cs = 0, clusters = 0;
  size_t smem = 0;
};
ScanLaunch g_cache;

}  // namespace

cudaError_t launch_scan(const Ctx& c, int m_max, cudaStream_t st) {
  // slice: multiple of 512 so CTAs own whole canonical chunks; <= 16 CTAs
  int slice = ((m_max + 15) / 16 + kChunk - 1) / kChunk * kChunk;
  if (slice < 1024) slice = 1024;
  if (slice > kMaxSlice / kChunk * kChunk) return cudaErrorInvalidValue;
  int cs = (m_max + slice - 1) / slice;
  if (cs < 1) cs = 1;
  const size_t smem = (size_t)(slice + 2) * 8 + 3 * (size_t)(slice / kChunk) * 8 + sizeof(Shared);
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
  if (g_cache.slice != slice || g_cache.cs != cs || g_cache.smem != smem) {
    cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cfg.gridDim = dim3(cs * 64, 1, 1);
    int clusters = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&clusters, scan_kernel, &cfg);
    if (e != cudaSuccess || clusters < 1) clusters = 148 / cs;
    if (clusters < 1) clusters = 1;
    g_cache = {slice, cs, clusters, smem};
  }
  const int n_items = 2 * c.NS;
  int clusters = g_cache.clusters;
  if (clusters > n_items) clusters = n_items;
  cfg.gridDim = dim3(cs * clusters, 1, 1);
  return cudaLaunchKernelEx(&cfg, scan_kernel, c, slice, n_items);
}

}  // namespace lfps
