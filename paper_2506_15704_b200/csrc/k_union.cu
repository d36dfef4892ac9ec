// k_union.cu -- the union of one (request, KV-head) unit's probe sets, for the
// per-unit finish (k_unit.cu, LFPS_FLAG_UNIT_FINISH).
//
// The G q-heads of a GQA unit share its K / V rows, and their probe sets
// (candidates.py:85-100, one per head) overlap by ~90%.  The per-unit finish
// streams every row of the union ONCE for all G heads; this kernel builds the
// table it streams, one 256-thread CTA per unit:
//
//   fused    when every non-gated head keeps its whole probe set (k >=
//            |probe|: C2 = probe, attention.py:34-47 -- the common case at
//            5%) the unit is fused: K / C2 counts are final here and each
//            head's probe list is copied to its C2 list; otherwise the count
//            is -1 and the per-session finish kernel (k_finish.cu) takes the
//            unit's sessions (the Top-k cut)
//   bitmaps  each head's sorted probe list is scattered into a per-head
//            bitmap of the context in shared memory (a window of 32 W rows
//            at a time; one window covers contexts up to n_max <= 256k), and
//            the words that hold a row into a presence bitmap
//   words    the active words (any head), in order, with one block scan of
//            their (union, head 0..3) popcounts: each gets its first union
//            position and each head's list rank at its first row
//   entries  a warp per active word, a lane per bit: the sinks first (every
//            non-gated head, no rank), then union row x = row | member
//            heads << 24 with the row's index in every member head's list
//            (its C2 rank), ascending -- balanced however the rows cluster
//            (the dense local tail, vertical bands)
#include "common.cuh"
#include "ptx.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUG = 4;                 // heads per unit (GQA group) this kernel serves
constexpr int kMaxWinW = 8192;         // bitmap words per head and window
constexpr int kAW = 1024;              // active words per pass

struct UnionShared {
  int p[kUG], byp[kUG];
  int red[kUG + 1][kWarps];
  int wsum[kWarps];
  int aw[kAW];                         // active word index
  int ab[kAW][kUG + 1];                // its first union position, first rank in each head
};

__host__ __device__ inline int union_win_words(int n_max) {
  const int w = (n_max + 31) / 32;
  return w < kMaxWinW ? w : kMaxWinW;
}

__global__ void __launch_bounds__(kThreads) lfps_union_kernel(Ctx c, int W) {
  extern __shared__ __align__(16) uint32_t bm[];   // [kUG][W] bitmaps, then [ceil(W / 32)] presence
  __shared__ UnionShared us;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* pres = bm + kUG * W;
  const int PW = (W + 31) >> 5;
  pdl_wait();                                   // the select kernel's lists and counts
  const int u = c.s_off / kUG + blockIdx.x;
  const int b = u / c.Hkv;
  const int n = c.n_ctx[b];
  const int S = c.S;
  if (tid < kUG) {
    const int sg = u * kUG + tid;
    us.byp[tid] = c.bypass[sg];
    us.p[tid] = c.counts[(size_t)sg * CNT_N + CNT_PROBE];
  }
  __syncthreads();
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  int hmask = 0, p[kUG];
  bool fused = true;
#pragma unroll
  for (int g = 0; g < kUG; ++g) {
    p[g] = us.byp[g] ? 0 : us.p[g];
    if (us.byp[g]) continue;
    hmask |= 1 << g;
    fused &= k >= us.p[g];
  }
  if (!fused) {
    if (tid == 0) c.unit_count[u] = -1;
    pdl_trigger();
    return;
  }
  if (tid < kUG) {                              // the counts the per-session finish would write
    int* cnt = c.counts + (size_t)(u * kUG + tid) * CNT_N;
    if (us.byp[tid]) { cnt[CNT_K] = 0; cnt[CNT_C2] = 0; cnt[CNT_CLAMP] = 0; }
    else { cnt[CNT_K] = k; cnt[CNT_C2] = us.p[tid]; }
  }
  if (!hmask) {
    if (tid == 0) c.unit_count[u] = 0;
    pdl_trigger();
    return;
  }
  int* ent = c.unit_ent + (size_t)u * c.unit_cap;
  int4* rnk = reinterpret_cast<int4*>(c.unit_rank) + (size_t)u * c.unit_cap;
  for (int j = tid; j < S; j += kThreads) {
    ent[j] = j | (hmask << 24) | (1 << 28);
    rnk[j] = make_int4(-1, -1, -1, -1);
  }
  int pos = S, rk0[kUG] = {0, 0, 0, 0};         // union position, list ranks at the pass start
#pragma unroll 1
  for (int R0 = 0; R0 < n; R0 += W * 32) {      // windows of W * 32 rows
    {
      uint4* z = reinterpret_cast<uint4*>(bm);
      const int nz = (kUG * W + PW + 3) >> 2;
      for (int i = tid; i < nz; i += kThreads) z[i] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
#pragma unroll
    for (int g = 0; g < kUG; ++g) {
      const int* lg = c.probe_idx + (size_t)(u * kUG + g) * c.list_cap;
      int* c2 = c.c2_idx + (size_t)(u * kUG + g) * c.list_cap;
      for (int i0 = tid; i0 < p[g]; i0 += 4 * kThreads) {
        int row[4];                             // four loads in flight before the atomics
#pragma unroll
        for (int q = 0; q < 4; ++q) row[q] = i0 + q * kThreads < p[g] ? __ldg(lg + i0 + q * kThreads) : -1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (row[q] < 0) continue;
          if (R0 == 0) c2[i0 + q * kThreads] = row[q];   // the C2 list (C2 = probe)
          const int x = row[q] - R0;
          if (x >= 0 && x < W * 32) {
            const int w = x >> 5;
            atomicOr(bm + g * W + w, 1u << (x & 31));
            atomicOr(pres + (w >> 5), 1u << (w & 31));
          }
        }
      }
    }
    __syncthreads();
    // ---- the active words in order, in passes of <= kAW ----------------------------------
#pragma unroll 1
    for (int pw0 = 0;;) {
      // presence words [pw0, pw1) holding <= kAW active words: thread t scans
      // presence word pw0 + t (PW <= 256 per pass at W <= 8192)
      const int pwi = pw0 + tid;
      const int cnt_t = pwi < PW ? __popc(pres[pwi]) : 0;
      int x = cnt_t;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(LFPS_FULL, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) us.wsum[warp] = x;
      __syncthreads();
      int before = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) before += w < warp ? us.wsum[w] : 0;
      const int start = before + x - cnt_t;     // active words before presence word pwi
      // this pass takes the presence words whose active words all fit below kAW
      const bool take = pwi < PW && start + cnt_t <= kAW;
      const int npw = __syncthreads_count(take);   // taken presence words: a prefix
      if (take) {
        int a = start;
        for (uint32_t m = pres[pwi]; m; m &= m - 1) us.aw[a++] = pwi * 32 + __ffs(m) - 1;
      }
      int na = 0;
      if (npw > 0) {
        // na = active words of the taken prefix (from the last taken thread)
        na = (int)__reduce_max_sync(LFPS_FULL, take ? start + cnt_t : 0);
      }
      if (lane == 0) us.wsum[warp] = na;
      __syncthreads();
      na = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) na = max(na, us.wsum[w]);
      // popcounts of the active words -> first positions (block scan, <= 4 words a thread)
      constexpr int kPer = kAW / kThreads;
      int v[kPer][kUG + 1];
      int tsum[kUG + 1] = {0, 0, 0, 0, 0};
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int a = tid * kPer + q;
        uint32_t uo = 0u;
#pragma unroll
        for (int g = 0; g < kUG; ++g) {
          const uint32_t hw = a < na ? bm[g * W + us.aw[a]] : 0u;
          uo |= hw;
          v[q][1 + g] = __popc(hw);
        }
        v[q][0] = __popc(uo);
#pragma unroll
        for (int i = 0; i <= kUG; ++i) tsum[i] += v[q][i];
      }
      int xs[kUG + 1];
#pragma unroll
      for (int i = 0; i <= kUG; ++i) xs[i] = tsum[i];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int i = 0; i <= kUG; ++i) {
          const int y = __shfl_up_sync(LFPS_FULL, xs[i], o);
          if (lane >= o) xs[i] += y;
        }
      }
      __syncthreads();                          // us.wsum reads above are done
      if (lane == 31) {
#pragma unroll
        for (int i = 0; i <= kUG; ++i) us.red[i][warp] = xs[i];
      }
      __syncthreads();
      int run[kUG + 1], total[kUG + 1];
#pragma unroll
      for (int i = 0; i <= kUG; ++i) {
        int bf = 0, tt = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
          const int t = us.red[i][w];
          bf += w < warp ? t : 0;
          tt += t;
        }
        run[i] = (i == 0 ? pos : rk0[i - 1]) + bf + xs[i] - tsum[i];
        total[i] = tt;
      }
#pragma unroll
      for (int q = 0; q < kPer; ++q) {
        const int a = tid * kPer + q;
        if (a < na) {
#pragma unroll
          for (int i = 0; i <= kUG; ++i) us.ab[a][i] = run[i];
        }
#pragma unroll
        for (int i = 0; i <= kUG; ++i) run[i] += v[q][i];
      }
      __syncthreads();
      // ---- entries: a warp per active word, a lane per bit -----------------------------
      const uint32_t lt = (1u << lane) - 1u;
      for (int a = warp; a < na; a += kWarps) {
        const int w = us.aw[a];
        uint32_t hw[kUG], uo = 0u;
#pragma unroll
        for (int g = 0; g < kUG; ++g) {
          hw[g] = bm[g * W + w];
          uo |= hw[g];
        }
        if (!((uo >> lane) & 1u)) continue;
        int mk = 0, r4[kUG];
#pragma unroll
        for (int g = 0; g < kUG; ++g) {
          const bool in = (hw[g] >> lane) & 1u;
          mk |= (int)in << g;
          r4[g] = in ? us.ab[a][1 + g] + __popc(hw[g] & lt) : -1;
        }
        const int at = us.ab[a][0] + __popc(uo & lt);
        ent[at] = (R0 + w * 32 + lane) | (mk << 24);
        rnk[at] = make_int4(r4[0], r4[1], r4[2], r4[3]);
      }
      pos += total[0];
#pragma unroll
      for (int g = 0; g < kUG; ++g) rk0[g] += total[1 + g];
      pw0 += npw;
      __syncthreads();                          // us.aw / us.ab are consumed
      if (pw0 >= PW || npw == 0) break;
    }
    __syncthreads();                            // the bitmaps are consumed
  }
  if (tid == 0) c.unit_count[u] = pos;
  pdl_trigger();
}

}  // namespace

cudaError_t launch_union(const Ctx& c, cudaStream_t st) {
  const int W = union_win_words(c.n_max);
  const size_t smem = ((size_t)kUG * W + (W + 31) / 32 + 3) / 4 * 16;
  static DeviceOnce once;
  cudaError_t e = once.run([] {
    return cudaFuncSetAttribute(lfps_union_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)(((size_t)kUG * kMaxWinW + kMaxWinW / 32 + 3) / 4 * 16));
  });
  if (e != cudaSuccess) return e;
  return launch_pdl(lfps_union_kernel, dim3(c.s_cnt / kUG), dim3(kThreads), smem, st, c, W);
}

}  // namespace lfps
