// k_tables.cu -- the tracker-table pipeline: moments (K1), thresholds,
// candidate bitmaps and the probe list (K2), in ONE persistent kernel.
//
// Every (session, table) item is cut into work units of 16384 slots (32
// canonical 512-slot chunks, four per warp).  Units of three phases flow
// through one statically scheduled queue:
//
//   A  one read of the phys table: per chunk the mean and centred power sums
//      M2, M3, M4; the item's last unit merges the chunks (exact pairwise
//      updates, canonical tree) into mean, s2, s4 and derives tau,
//      mean/scale and the degenerate flag (tables.py:127-140, 295-317)
//   B  ballot bitmaps  C0 = phys > tau/scale  (select_initial, candidates.py:45-58)
//                      F  = phys > mean/scale (expand's filter, candidates.py:79-81)
//   C  per session: C1 = F & dilate(C0), probe = C1 | local window, sorted
//      index list (expand + finalize_probe_set, candidates.py:61-100)
//
// The queue is skewed by "waves" of items -- slot k holds A(wave k),
// B(wave k-2), C(wave k-4) -- so B's re-read of a table finds it in L2 (the
// window of three waves is sized to ~48 MB of the 126 MB L2) and every table
// byte crosses HBM once.  Dependencies are counters/flags in global memory
// and always point to earlier queue positions; each CTA walks its positions
// in order, so the persistent grid cannot deadlock.
//
// Arithmetic is the canonical devmath.table_moments (chunk = 512 slots,
// lane l holds slots e*32 + l, adjacent-pair trees over e, lane folds, then a
// pairwise merge tree over all chunks), bit-identical to the oracle and
// independent of unit / wave sizes.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 512;
constexpr int kChunksPerWarp = 1;
constexpr int kUnitChunks = kWarps * kChunksPerWarp;   // 32 chunks
constexpr int kUnit = kChunk * kUnitChunks;            // 16384 slots (128 KB)
constexpr int kTreeLeaves = 512;             // chunks per table: m <= 262144
constexpr int kLeavesPerLane = kTreeLeaves / 32;

// per-item counters / flags (int) and scalars (double) in the workspace
enum { CT_A = 0, CT_B, CT_READY, CT_N = 4 };
enum { IF_THR0 = 0, IF_THRF, IF_DEG, IF_N = 4 };
enum { PH_A = 0, PH_B = 1, PH_C = 2 };
constexpr int kSkewB = 2;   // B(wave k - 2) sits in slot k
constexpr int kSkewC = 4;   // C(wave k - 4) sits in slot k

// Round schedule: in round r, CTA j does A unit r*G + j, then B unit
// (r - kLagB)*G + j, then (maybe) the probe list of one session whose B units
// all belong to rounds <= r - kLagC.  Dependencies point >= 2 rounds back;
// the L2 must hold ~kLagB rounds of A data (G x 32 KB per round).
constexpr int kLagB = 3;
constexpr int kLagC = 2;   // rounds after a session's last B unit
struct Sched {
  int n_items, U, G, rounds;
  long long na;            // A (and B) units = n_items * U
};

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void spin_until_ge(const int* p, int target) {
  while (ld_acquire(p) < target) __nanosleep(64);
}

// 16 slots of chunk `ch` for this lane: logical e*32 + lane (masked to 0)
__device__ __forceinline__ void load_chunk(const Ctx& c, int s, int table, int base, int m, int ch,
                                           int lane, double* v) {
  const int i0 = ch * kChunk;
  if (table == 0) {
    const double* src = c.ver + (size_t)s * c.m_cap + i0 + lane;
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = (i0 + e * 32 + lane < m) ? src[e * 32] : 0.0;
  } else {
    const int C = c.ring_cap;
    const double* ring = c.sla + (size_t)s * C;
    int p0 = (base + i0) % C;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      int p = p0 + e * 32 + lane;
      if (p >= C) p -= C;
      v[e] = (i0 + e * 32 + lane < m) ? ring[p] : 0.0;
    }
  }
}

__device__ __forceinline__ double tree16(double* v) {
#pragma unroll
  for (int h = 1; h < 16; h <<= 1) {
#pragma unroll
    for (int k = 0; k < 16; k += 2 * h) v[k] = cadd(v[k], v[k + h]);
  }
  return v[0];
}

__device__ __forceinline__ long long thr_bits(double t) {
  return isnan(t) ? 0x7fffffffffffffffll : __double_as_longlong(t);
}

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
  const double dn = cdiv(delta, r.n);
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

struct Pipe {
  double* part;   // [n_items][4][kTreeLeaves]: chunk mean, M2, M3, M4
  double* itemf;  // [n_items][IF_N]
  int* ctr;       // [n_items][CT_N]
  int* work;      // [1]
};

// canonical merge tree over the item's chunk moments (zero-count padding to
// kTreeLeaves); lane l owns leaves [16 l, 16 l + 16); all lanes return it
__device__ __noinline__ Mom merge_tree(const double* part, int n_chunks, int m, int lane) {
  // in-lane adjacent-pair tree over 16 leaves, streamed through a 4-level
  // stack (level l holds a pending left subtree of 2^l leaves)
  Mom stk[4];
  Mom cur;
#pragma unroll
  for (int k = 0; k < kLeavesPerLane; ++k) {
    const int i = lane * kLeavesPerLane + k;
    cur = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (i < n_chunks) {
      cur.n = (double)min(kChunk, m - i * kChunk);
      cur.mu = __ldcg(part + i);
      cur.m2 = __ldcg(part + kTreeLeaves + i);
      cur.m3 = __ldcg(part + 2 * kTreeLeaves + i);
      cur.m4 = __ldcg(part + 3 * kTreeLeaves + i);
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
  Mom acc = cur;   // after k = 15 every level has merged: the 16-leaf tree
#pragma unroll
  for (int h = 1; h <= 16; h <<= 1) {
    const Mom o = shfl_mom(acc, h);
    acc = (lane & h) ? merge(o, acc) : merge(acc, o);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// Phase C: probe list for session s (bits of both tables complete)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t shifted(uint32_t prev, uint32_t cur, uint32_t next, int delta) {
  if (delta == 0) return cur;
  if (delta > 0) return (cur << delta) | (prev >> (32 - delta));
  const int k = -delta;
  return (cur >> k) | (next << (32 - k));
}

__device__ void phase_c(const Ctx& c, int s, int m, uint32_t* pwords, int* blk, int (*red)[kWarps]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* cnt = c.counts + (size_t)s * CNT_N;
  const int S = c.S;
  const int W = (m + 31) / 32;
  const int nblk = (W + 31) / 32;
  const uint32_t* c0v = c.bits + ((size_t)(s * 2 + 0) * 2 + 0) * c.words;
  const uint32_t* fv = c.bits + ((size_t)(s * 2 + 0) * 2 + 1) * c.words;
  const uint32_t* c0s = c.bits + ((size_t)(s * 2 + 1) * 2 + 0) * c.words;
  const uint32_t* fs = c.bits + ((size_t)(s * 2 + 1) * 2 + 1) * c.words;
  const int tail_lo = max(0, m - c.L);
  const uint32_t last_valid = (m & 31) ? ((1u << (m & 31)) - 1u) : LFPS_FULL;
  int n0 = 0, n1 = 0, nd = 0;
  for (int bk = warp; bk < nblk; bk += kWarps) {
    const int w = bk * 32 + lane;
    const bool in = w < W;
    const uint32_t cur = in ? (__ldcg(c0v + w) | __ldcg(c0s + w)) : 0u;
    const uint32_t f = in ? (__ldcg(fv + w) | __ldcg(fs + w)) : 0u;
    uint32_t prev = __shfl_up_sync(LFPS_FULL, cur, 1);
    uint32_t next = __shfl_down_sync(LFPS_FULL, cur, 1);
    if (lane == 0) prev = (w > 0 && w - 1 < W) ? (__ldcg(c0v + w - 1) | __ldcg(c0s + w - 1)) : 0u;
    if (lane == 31) next = (w + 1 < W) ? (__ldcg(c0v + w + 1) | __ldcg(c0s + w + 1)) : 0u;
    uint32_t dil = 0;
    for (int k = 0; k < c.n_off; ++k) dil |= shifted(prev, cur, next, c.off[k]);
    const uint32_t valid = !in ? 0u : (w == W - 1 ? last_valid : LFPS_FULL);
    const uint32_t c1 = f & dil & valid;
    uint32_t tail = 0;
    const int j0 = w * 32;
    if (in && j0 + 32 > tail_lo) tail = (LFPS_FULL << max(0, tail_lo - j0)) & valid;
    const uint32_t pr = c1 | tail;
    if (in) pwords[w] = pr;
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
    for (int base = 0; base < nblk; base += 32) {
      const int i = base + lane;
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

// first session whose probe list is scheduled in round >= r
__device__ __forceinline__ int c_first(const Sched& sc, int r) {
  // probe of session s waits for B unit (2s+2)U-1, which runs in round
  // ((2s+2)U-1)/G + kLagB; it is scheduled kLagC rounds later
  const long long t = (long long)sc.G * (r - kLagB - kLagC) + 1;
  if (t <= 0) return 0;
  const long long s = (t + 2LL * sc.U - 1) / (2LL * sc.U) - 1;
  return (int)(s < 0 ? 0 : s);
}

__global__ void __launch_bounds__(kThreads, 3) tables_kernel(Ctx c, Pipe pp, Sched sc) {
  extern __shared__ uint32_t pwords[];           // phase C scratch
  __shared__ int blk[192];
  __shared__ int red[4][kWarps];
  __shared__ int sh_flag;
  __shared__ double sh_d[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n_sessions = sc.n_items / 2;

  for (int rnd = 0; rnd < sc.rounds; ++rnd) {
    for (int phase = PH_A; phase <= PH_C; ++phase) {
      int item = 0, u = 0;
      if (phase == PH_C) {
        const int s = c_first(sc, rnd) + blockIdx.x;
        if (s >= c_first(sc, rnd + 1) || s >= n_sessions) continue;
        const int m = c.n_ctx[s / c.Hq] - c.S;
        if (c.bypass[s]) {
          if (tid < CNT_N) c.counts[(size_t)s * CNT_N + tid] = 0;
          continue;
        }
        const int Us = (m + kUnit - 1) / kUnit;
        if (tid == 0) {
          spin_until_ge(pp.ctr + (size_t)(2 * s) * CT_N + CT_B, Us);
          spin_until_ge(pp.ctr + (size_t)(2 * s + 1) * CT_N + CT_B, Us);
          __threadfence();
        }
        __syncthreads();
        phase_c(c, s, m, pwords, blk, red);
        __syncthreads();
        continue;
      }
      const long long unit = (long long)(rnd - (phase == PH_A ? 0 : kLagB)) * sc.G + blockIdx.x;
      if (unit < 0 || unit >= sc.na) continue;
      item = (int)(unit / sc.U);
      u = (int)(unit % sc.U);
      const int s = item >> 1, table = item & 1;
      if (c.bypass[s]) continue;
      const int m = c.n_ctx[s / c.Hq] - c.S;
      const int Us = (m + kUnit - 1) / kUnit;
      if (u >= Us) continue;
      const int base = table ? c.sla_base[s] : 0;
      const int ch0 = u * kUnitChunks + warp;      // warp's chunks: ch0 + j * kWarps
      const int n_chunks = (m + kChunk - 1) / kChunk;
      int* ctr = pp.ctr + (size_t)item * CT_N;
      double* itemf = pp.itemf + (size_t)item * IF_N;
      double* part = pp.part + (size_t)item * 4 * kTreeLeaves;
      if (phase == PH_A) {
        if (c.exhaustive) continue;
        for (int j = 0; j < kChunksPerWarp; ++j) {
          const int ch = ch0 + j * kWarps;
          if (ch >= n_chunks) break;
          double v[16];
          load_chunk(c, s, table, base, m, ch, lane, v);   // invalid slots read as 0
          const int i0 = ch * kChunk;
          const double cnt = (double)min(kChunk, m - i0);
          // chunk mean: adjacent-pair tree over e, lane fold, / count
          double q[4];
  #pragma unroll
          for (int gq = 0; gq < 4; ++gq)
            q[gq] = cadd(cadd(v[4 * gq], v[4 * gq + 1]), cadd(v[4 * gq + 2], v[4 * gq + 3]));
          const double mu = cdiv(warp_fold(cadd(cadd(q[0], q[1]), cadd(q[2], q[3]))), cnt);
          // centred powers d^2, d^3, d^4 in the same tree order
          double p2[4], p3[4], p4[4];
  #pragma unroll
          for (int gq = 0; gq < 4; ++gq) {
            double t2[4], t3[4], t4[4];
  #pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int e = 4 * gq + t;
              const double d = (i0 + e * 32 + lane < m) ? csub(v[e], mu) : 0.0;
              const double d2 = cmul(d, d);
              t2[t] = d2;
              t3[t] = cmul(d2, d);
              t4[t] = cmul(d2, d2);
            }
            p2[gq] = cadd(cadd(t2[0], t2[1]), cadd(t2[2], t2[3]));
            p3[gq] = cadd(cadd(t3[0], t3[1]), cadd(t3[2], t3[3]));
            p4[gq] = cadd(cadd(t4[0], t4[1]), cadd(t4[2], t4[3]));
          }
          const double m2 = warp_fold(cadd(cadd(p2[0], p2[1]), cadd(p2[2], p2[3])));
          const double m3 = warp_fold(cadd(cadd(p3[0], p3[1]), cadd(p3[2], p3[3])));
          const double m4 = warp_fold(cadd(cadd(p4[0], p4[1]), cadd(p4[2], p4[3])));
          if (lane == 0) {
            part[ch] = mu;
            part[kTreeLeaves + ch] = m2;
            part[2 * kTreeLeaves + ch] = m3;
            part[3 * kTreeLeaves + ch] = m4;
          }
        }
        if (lane == 0) __threadfence();
        __syncthreads();
        if (tid == 0) {
          __threadfence();
          sh_flag = atomicAdd(ctr + CT_A, 1) == Us - 1;
        }
        __syncthreads();
        if (sh_flag && warp == 0) {          // last unit: merge -> thresholds
          __threadfence();
          const Mom tot = merge_tree(part, n_chunks, m, lane);
          if (lane == 0) {
            const double scl = c.scale[s];
            const double mean_p = tot.mu, s2p = tot.m2, s4p = tot.m4;
            const double mean = cmul(mean_p, scl);
            const bool deg = cmul(cmul(s2p, scl), scl) < 1e-12;
            double tau = NAN, kappa = NAN, thr0 = NAN;
            if (!deg) {
              kappa = cdiv(s4p, cmul(s2p, s2p));
              if (kappa == 0.0) set_err(c, s, LFPS_ERR_KAPPA_ZERO);
              tau = cdiv(cmul(c.a, mean), kappa);
              thr0 = cdiv(tau, scl);
            }
            itemf[IF_THR0] = thr0;
            itemf[IF_THRF] = cdiv(mean, scl);
            itemf[IF_DEG] = deg ? 1.0 : 0.0;
            double* thr = c.thr + (size_t)item * 4;
            thr[0] = tau; thr[1] = mean; thr[2] = deg ? 1.0 : 0.0; thr[3] = kappa;
            __threadfence();
            atomicExch(ctr + CT_READY, 1);
          }
        }
        __syncthreads();
        continue;
      }


      // ---- PH_B: bitmaps (the table is re-read from L2) ----
      long long tb0, tbf;
      if (c.exhaustive) {
        tb0 = tbf = -1ll;      // every valid phys value (>= +0) passes
        if (u == 0 && tid == 0) {
          double* thr = c.thr + (size_t)item * 4;
          thr[0] = -INFINITY; thr[1] = -INFINITY; thr[2] = 0.0; thr[3] = NAN;
        }
      } else {
        if (tid == 0) {
          spin_until_ge(ctr + CT_READY, 1);
          __threadfence();
          sh_d[1] = __ldcg(itemf + IF_THR0);
          sh_d[2] = __ldcg(itemf + IF_THRF);
          sh_d[3] = __ldcg(itemf + IF_DEG);
        }
        __syncthreads();
        tb0 = sh_d[3] != 0.0 ? 0x7fffffffffffffffll : thr_bits(sh_d[1]);
        tbf = thr_bits(sh_d[2]);
      }
      for (int j = 0; j < kChunksPerWarp; ++j) {
        const int ch = ch0 + j * kWarps;
        if (ch >= n_chunks) break;
        double v[16];
        if (!c.exhaustive) load_chunk(c, s, table, base, m, ch, lane, v);
        const int i0 = ch * kChunk;
        uint32_t my = 0;
  #pragma unroll
        for (int e = 0; e < 16; ++e) {
          const bool ok = i0 + e * 32 + lane < m;
          const long long x = c.exhaustive ? 0ll : __double_as_longlong(v[e]);
          const uint32_t w0 = __ballot_sync(LFPS_FULL, ok && x > tb0);
          const uint32_t wf = __ballot_sync(LFPS_FULL, ok && x > tbf);
          if (lane == e) my = w0;
          if (lane == 16 + e) my = wf;
        }
        uint32_t* bits = c.bits + ((size_t)item * 2 + (lane >> 4)) * c.words;
        bits[ch * 16 + (lane & 15)] = my;
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicAdd(ctr + CT_B, 1);

    }
  }
}

__global__ void tables_reset_kernel(int* ctr, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    ctr[i] = 0;
}

size_t g_grid_smem = 0;
int g_grid = 0;

}  // namespace

size_t tables_pipe_bytes(int n_items) {
  return (size_t)n_items * (4 * kTreeLeaves + IF_N) * 8 + (size_t)n_items * CT_N * 4 + 256;
}

cudaError_t launch_tables(const Ctx& c, void* pipe_base, int m_max, cudaStream_t st) {
  if ((m_max + kChunk - 1) / kChunk > kTreeLeaves) return cudaErrorInvalidValue;
  const int n_items = 2 * c.NS;
  Pipe pp;
  char* b = static_cast<char*>(pipe_base);
  pp.part = reinterpret_cast<double*>(b);
  pp.itemf = pp.part + (size_t)n_items * 4 * kTreeLeaves;
  pp.ctr = reinterpret_cast<int*>(pp.itemf + (size_t)n_items * IF_N);
  pp.work = pp.ctr + (size_t)n_items * CT_N;
  const size_t smem = (size_t)c.words * 4;
  if (!g_grid || g_grid_smem != smem) {
    g_grid_smem = smem;
    cudaFuncSetAttribute(tables_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tables_kernel, kThreads, smem);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g_grid = sms * (per_sm > 0 ? per_sm : 1);
  }
  Sched sc;
  sc.n_items = n_items;
  sc.U = (m_max + kUnit - 1) / kUnit;
  if (sc.U < 1) sc.U = 1;
  sc.na = (long long)n_items * sc.U;
  sc.G = g_grid;
  if (sc.na < sc.G) sc.G = (int)sc.na;
  sc.rounds = (int)((sc.na + sc.G - 1) / sc.G) + kLagB + kLagC + 2;
  tables_reset_kernel<<<64, 256, 0, st>>>(pp.ctr, (size_t)n_items * CT_N + 2);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  tables_kernel<<<sc.G, kThreads, smem, st>>>(c, pp, sc);
  return cudaGetLastError();
}

}  // namespace lfps
