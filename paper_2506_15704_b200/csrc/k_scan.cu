// k_scan.cu -- tracker-table scan (K1 moments + the threshold half of K2).
//
// One thread-block cluster per (session, table).  Each CTA owns a contiguous
// slice of the table's logical range, pulls it into shared memory ONCE with
// 1-D bulk async copies (cp.async.bulk, mbarrier completion), and then runs
// every pass from shared memory:
//
//   pass 1  chunk sums            -> cluster-wide mean  (DSMEM gather)
//   pass 2  centred c^2, c^4 sums -> cluster-wide s2, s4 (DSMEM gather)
//   thresholds tau / mean / degenerate (tables.py:295-317)
//   pass 3  ballot bitmaps: C0 bit = phys > tau/scale (select_initial,
//           candidates.py:45-58), F bit = phys > mean/scale (the expansion
//           filter, candidates.py:79-81); written to the workspace.
//
// The HBM traffic is the table itself (8 B per slot), read once; the two
// bitmaps written are 1/32 of it.  Summation order is canonical
// (devmath.table_sum): 512-element warp chunks, lane-strided, folded, then a
// pairwise tree over all chunk partials of the session, so the result does
// not depend on how many CTAs the cluster has.
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

__global__ void __launch_bounds__(kThreads) scan_kernel(Ctx c, int slice) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* data = reinterpret_cast<double*>(smem_raw);                 // [slice + 2]
  double* part1 = data + slice + 2;                                    // [slice / 512]
  double* part2 = part1 + slice / kChunk;
  double* part4 = part2 + slice / kChunk;
  Shared* sh = reinterpret_cast<Shared*>(part4 + slice / kChunk);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = blockIdx.y >> 1, table = blockIdx.y & 1;
  if (c.bypass[s]) return;                       // uniform across the cluster
  const int b = s / c.Hq;
  const int m = c.n_ctx[b] - c.S;
  const uint32_t rank = cluster_rank();
  const int lo = (int)rank * slice;
  const int cnt = max(0, min(slice, m - lo));
  const int cpc = slice / kChunk;                // chunks per CTA
  const int words_cta = slice / 32;
  uint32_t* bits_c0 = c.bits + ((size_t)(s * 2 + table) * 2 + 0) * c.words;
  uint32_t* bits_f = c.bits + ((size_t)(s * 2 + table) * 2 + 1) * c.words;

  if (c.exhaustive) {
    // thresholds and means are -inf (engine.py:29-32): every valid slot is
    // in C0 and passes the filter; no table bytes are needed.
    for (int w = tid; w < words_cta; w += kThreads) {
      const int i0 = w * 32;
      const int valid = max(0, min(32, cnt - i0));
      const uint32_t word = valid == 32 ? LFPS_FULL : ((1u << valid) - 1u);
      bits_c0[lo / 32 + w] = word;
      bits_f[lo / 32 + w] = word;
    }
    if (rank == 0 && tid == 0) {
      double* thr = c.thr + (size_t)(s * 2 + table) * 4;
      thr[0] = -INFINITY; thr[1] = -INFINITY; thr[2] = 0.0; thr[3] = NAN;
    }
    return;
  }

  // ---- stage the slice into shared memory --------------------------------
  const double* src_ver = c.ver + (size_t)s * c.m_cap;
  const double* src_sla = c.sla + (size_t)s * c.ring_cap;
  const int C = c.ring_cap;
  const int base = c.sla_base[s];
  // smem element e <-> logical (lo - off + e); off keeps the copy 16B aligned
  int off = 0;
  if (table == 1) off = ((base + lo) % C) & 1;
  const int total = cnt > 0 ? ((off + cnt + 1) & ~1) : 0;   // even element count
  const int nst = (total + kStage - 1) / kStage;
  if (tid == 0) {
    for (int j = 0; j < nst; ++j) mbar_init(&sh->bar[j], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    for (int j = 0; j < nst; ++j) {
      const int e0 = j * kStage;
      const int len = min(kStage, total - e0);
      mbar_expect_tx(&sh->bar[j], (uint32_t)len * 8u);
      const int logical = lo - off + e0;
      if (table == 0) {
        bulk_g2s(data + e0, src_ver + logical, (uint32_t)len * 8u, &sh->bar[j]);
      } else {
        const int p = ((base + logical) % C + C) % C;
        const int first = min(len, C - p);
        bulk_g2s(data + e0, src_sla + p, (uint32_t)first * 8u, &sh->bar[j]);
        if (first < len)
          bulk_g2s(data + e0 + first, src_sla, (uint32_t)(len - first) * 8u, &sh->bar[j]);
      }
    }
  }

  // ---- pass 1: chunk sums ---------------------------------------------------
  for (int ch = warp; ch < cpc; ch += kWarps) {
    const int i0 = ch * kChunk;
    const int vc = max(0, min(kChunk, cnt - i0));
    double acc = 0.0;
    if (vc > 0) {
      mbar_wait(&sh->bar[(off + i0) / kStage], 0);
      mbar_wait(&sh->bar[(off + i0 + vc - 1) / kStage], 0);
#pragma unroll 4
      for (int e = 0; e < kChunk / 32; ++e) {
        const int i = i0 + e * 32 + lane;
        if (i < cnt) acc = cadd(acc, data[off + i]);
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
#pragma unroll 4
      for (int e = 0; e < kChunk / 32; ++e) {
        const int i = i0 + e * 32 + lane;
        if (i < cnt) {
          const double x = csub(data[off + i], mean_p);
          const double x2 = cmul(x, x);
          a2 = cadd(a2, x2);
          a4 = cadd(a4, cmul(x2, x2));
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
  // every remote read of this cluster's partials is done once all CTAs arrive
  cluster_arrive();

  // ---- thresholds (tables.py:305-317, candidates.py:52-54) ------------------
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

  // ---- pass 3: ballot bitmaps ----------------------------------------------
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
  cluster_wait();
}

}  // namespace

static int g_scan_smem_set = 0;

cudaError_t launch_scan(const Ctx& c, int m_max, cudaStream_t st) {
  // slice: multiple of 512 so CTAs own whole canonical chunks; <= 16 CTAs
  int slice = ((m_max + 15) / 16 + kChunk - 1) / kChunk * kChunk;
  if (slice < 1024) slice = 1024;
  if (slice > kMaxSlice / kChunk * kChunk) return cudaErrorInvalidValue;
  int cs = (m_max + slice - 1) / slice;
  if (cs < 1) cs = 1;
  const size_t smem = (size_t)(slice + 2) * 8 + 3 * (size_t)(slice / kChunk) * 8 + sizeof(Shared);
  if (!g_scan_smem_set) {
    cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(scan_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    g_scan_smem_set = 1;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs, 2 * c.NS, 1);
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
  return cudaLaunchKernelEx(&cfg, scan_kernel, c, slice);
}

}  // namespace lfps
