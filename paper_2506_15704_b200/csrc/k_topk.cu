// k_topk.cu -- exact-path Top-k over every non-sink score of a session (KX).
//
// Restates topk_from_scores (attention.py:34-47) applied to the full score
// vector of exact_topk_step (bench.py:73-80), with the budget rule of
// decode_step (engine.py:167): k = max(1, round_half_even(frac * n)).  If
// k >= m every non-sink row is selected; otherwise the selection is
// {z > kth} plus the lowest-index entries with z == kth, emitted in index
// order.  Keys are order-preserving uint32 maps of the fp32 scores with -0.0
// canonicalised to +0.0 (canon.cuh score_key).  One 512-thread CTA per
// session; the m scores (512 KiB at 128k) are streamed ONCE:
//
//   0  a strided sample of 4096 keys; its order statistics at ranks around
//      k m / 4096 (+- 4 sqrt(rank) + 16), found by two radix selects in
//      shared memory (not a full sort), bound a key window
//      [lo, hi] that holds the k-th largest key with overwhelming probability;
//   1  one pass appends the (score, index) pairs above hi to a global
//      buffer (the session's uw scratch) and the window's to shared memory,
//      warp-aggregated;
//   2  if the window provably holds the k-th key (keys above hi < k <=
//      keys above hi + window size, and the window fit), an MSB-first radix
//      select over the window finds it exactly (ties: a second radix select
//      over the tied entries' indices finds the lowest need_eq of them);
//   3  the selected indices are set in a bitmap of the session's rows, the
//      bitmap's word prefixes give every selection its output position in
//      index order, and each selected pair is written there.
// If the window misses, the kernel falls back to a 2048-bin histogram pass
// over all keys, the same select on the k-th bin, and an ordered emission
// pass in which every warp re-walks its index chunk.  Loads are float4 (4
// keys per lane) with four in flight.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kSample = 4096;
constexpr int kBins = 2048;                 // fallback: top 11 key bits
constexpr int kShift = 21;
constexpr int kCand = 6144;                 // window candidates kept in shared memory

struct TopkShared {
  unsigned samp[kSample];                   // fallback histogram (kBins <= kSample); tie scratch
  uint2 cand[kCand];                        // window: (score bits, index); fallback: (key, index)
  int wsum[kWarps];
  int above[kWarps];                        // keys above the window, per warp chunk
  int gtc[kWarps], eqc[kWarps];             // window keys > kth / == kth, per warp chunk
  int ncand, over, nabove, neq;
  unsigned hist[256];
  unsigned sel_digit;
  int sel_want;
};

__device__ __forceinline__ uint32_t key_at(const float* z, int j) { return score_key(z[j]); }

// MSB-first radix select over keys[0, nk) restricted to (key & mask) ==
// prefix: the key value whose descending rank contains `want` (1-based),
// i.e. the want-th largest; returns it and sets *need_eq to how many keys
// equal to it are still to be taken.
template <typename KeyOf>
__device__ uint32_t radix_select(TopkShared& sh, const uint2* keys, int nk, uint32_t prefix,
                                 uint32_t mask, int first_shift, int want, int* need_eq, KeyOf key_of) {
  const int tid = threadIdx.x;
  for (int shift = first_shift; shift >= 0; shift -= 8) {
    if (tid < 256) sh.hist[tid] = 0;
    __syncthreads();
    for (int i = tid; i < nk; i += kThreads) {
      const uint32_t key = key_of(keys[i]);
      if ((key & mask) == prefix) atomicAdd(&sh.hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) {
      unsigned loc = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) loc += sh.hist[255 - 8 * tid - t];
      unsigned incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(LFPS_FULL, incl, o);
        if (tid >= o) incl += y;
      }
      const unsigned excl = incl - loc;
      if (excl < (unsigned)want && incl >= (unsigned)want) {
        unsigned cum = excl;
        for (int t = 0; t < 8; ++t) {
          const unsigned dgt = 255 - 8 * tid - t;
          const unsigned hc = sh.hist[dgt];
          if (cum + hc >= (unsigned)want) {
            sh.sel_digit = dgt;
            sh.sel_want = want - (int)cum;
            break;
          }
          cum += hc;
        }
      }
    }
    __syncthreads();
    prefix |= sh.sel_digit << shift;
    mask |= 255u << shift;
    want = sh.sel_want;
    __syncthreads();
  }
  *need_eq = want;
  return prefix;
}
__device__ __forceinline__ uint32_t key_x(uint2 e) { return e.x; }
__device__ __forceinline__ uint32_t key_bits(uint2 e) { return score_key(__uint_as_float(e.x)); }


__global__ void __launch_bounds__(kThreads) lfps_exact_topk_kernel(Ctx c) {
  extern __shared__ uint8_t dyn[];
  TopkShared& sh = *reinterpret_cast<TopkShared*>(dyn);
  const int s = blockIdx.x, tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  int* cnt = c.counts + (size_t)s * CNT_N;
  const int b = s / c.Hq;
  const int n = c.n_ctx[b];
  const int S = c.S;
  const int p = cnt[CNT_PROBE];                    // = m, set by the score kernel
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  const float* z = c.probe_score + (size_t)s * c.list_cap;
  int* out_i = c.c2_idx + (size_t)s * c.list_cap;
  float* out_z = c.c2_score + (size_t)s * c.list_cap;
  if (tid == 0) cnt[CNT_K] = k;
  if (k >= p) {
    for (int j = tid; j < p; j += kThreads) {
      out_i[j] = S + j;
      out_z[j] = z[j];
    }
    if (tid == 0) cnt[CNT_C2] = p;
    return;
  }
  // warp chunks: multiples of 128 keys (float4 per lane), the last one short
  const int chunk = ((p + kWarps - 1) / kWarps + 127) / 128 * 128;
  const int j0 = min(p, warp * chunk), j1 = min(p, j0 + chunk);
  const bool vec_ok = (reinterpret_cast<uintptr_t>(z) & 15) == 0;

  // ---- 0: sorted sample -> key window [lo, hi] -----------------------------------
  uint32_t lo = 0, hi = 0xffffffffu;
  bool use_window = p > 4 * kSample;
  if (use_window) {
    // the two sample order statistics by radix select (the sample is staged
    // as (key, i) in the candidate buffer, idle until pass 1)
    for (int i = tid; i < kSample; i += kThreads)
      sh.cand[i] = make_uint2(key_at(z, (int)(((long long)i * p) / kSample)), (uint32_t)i);
    __syncthreads();
    const int r = (int)(((long long)k * kSample) / p);
    const int delta = 4 * (int)sqrtf((float)r + 1.0f) + 16;
    const int rh = r - delta, rl = r + delta;
    int dummy;
    // (sorted descending, sample entry q would be the (q + 1)-th largest key)
    hi = rh <= 0 ? 0xffffffffu : radix_select(sh, sh.cand, kSample, 0u, 0u, 24, rh + 1, &dummy, key_x);
    lo = rl >= kSample ? 0u : radix_select(sh, sh.cand, kSample, 0u, 0u, 24, rl + 1, &dummy, key_x);
    if (tid == 0) { sh.ncand = 0; sh.over = 0; sh.nabove = 0; sh.neq = 0; }
    __syncthreads();
  }

  // ---- 1: the pairs above the window (global buffer) and in it (shared) -----------------
  uint2* abuf = reinterpret_cast<uint2*>(c.uw + (size_t)s * c.list_cap);   // list_cap pairs
  if (use_window) {
    // per lane 16 keys a round: the flags as bit masks, one warp scan of both
    // counts and one atomic per buffer and warp
    auto round = [&](const float (&zv)[16], const int (&jv)[16], int nok) {
      uint32_t ma = 0u, mw = 0u;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint32_t key = score_key(zv[i]);
        const bool ok = i < nok;
        ma |= (uint32_t)(ok && key > hi) << i;
        mw |= (uint32_t)(ok && key <= hi && key >= lo) << i;
      }
      const int cnt = __popc(ma) | (__popc(mw) << 16);
      int x = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(LFPS_FULL, x, o);
        if (lane >= o) x += y;
      }
      const int tot = __shfl_sync(LFPS_FULL, x, 31);
      if (!tot) return;
      int base = 0;
      if (lane == 0 && (tot & 0xffff)) base = atomicAdd(&sh.nabove, tot & 0xffff);
      if (lane == 1 && (tot >> 16)) base = atomicAdd(&sh.ncand, tot >> 16);
      const int ba = __shfl_sync(LFPS_FULL, base, 0) + ((x - cnt) & 0xffff);
      const int bw = __shfl_sync(LFPS_FULL, base, 1) + ((x - cnt) >> 16);
      // (static indices keep zv / jv in registers)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const uint2 e = make_uint2(__float_as_uint(zv[i]), (uint32_t)jv[i]);
        if ((ma >> i) & 1) abuf[ba + __popc(ma & ((1u << i) - 1u))] = e;
        const int at = bw + __popc(mw & ((1u << i) - 1u));
        if (((mw >> i) & 1) && at < kCand) sh.cand[at] = e;
      }
    };
    if (vec_ok) {
      // four float4 loads (16 keys) in flight per lane
      for (int base0 = j0; base0 < j1; base0 += 512) {
        float zv[16];
        int jv[16];
        int nok = 16;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int base = base0 + 128 * u + 4 * lane;
          float4 v;
          if (base + 3 < j1) {
            v = __ldg(reinterpret_cast<const float4*>(z + base));
          } else {
            v = make_float4(base < j1 ? z[base] : 0.f, base + 1 < j1 ? z[base + 1] : 0.f,
                            base + 2 < j1 ? z[base + 2] : 0.f, 0.f);
            if (nok == 16) nok = 4 * u + max(0, min(4, j1 - base));
          }
          zv[4 * u] = v.x; zv[4 * u + 1] = v.y; zv[4 * u + 2] = v.z; zv[4 * u + 3] = v.w;
#pragma unroll
          for (int e = 0; e < 4; ++e) jv[4 * u + e] = base + e;
        }
        round(zv, jv, nok);
      }
    } else {
      for (int b0 = j0; b0 < j1; b0 += 32 * 16) {
        float zv[16];
        int jv[16];
        int nok = 16;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = b0 + 32 * i + lane;
          zv[i] = j < j1 ? z[j] : 0.f;
          jv[i] = j;
          if (j >= j1 && nok == 16) nok = i;
        }
        round(zv, jv, nok);
      }
    }
  }
  if (lane == 0) { sh.gtc[warp] = 0; sh.eqc[warp] = 0; }
  __syncthreads();
  const int tot_above = use_window ? sh.nabove : 0;
  const int nc = use_window ? sh.ncand : 0;
  // the window provably holds the k-th key?
  use_window = use_window && nc <= kCand && tot_above < k && tot_above + nc >= k;

  if (use_window) {
    // ---- 2: the k-th key in the window; ties by lowest index ---------------------------
    int need_eq;
    const uint32_t kth = radix_select(sh, sh.cand, nc, 0u, 0u, 24, k - tot_above, &need_eq, key_bits);
    uint2* eqs = reinterpret_cast<uint2*>(sh.samp);            // kSample / 2 tied entries
    for (int i = tid; i < nc; i += kThreads) {
      const uint2 e = sh.cand[i];
      if (key_bits(e) == kth) {
        const int at = atomicAdd(&sh.neq, 1);
        if (at < kSample / 2) eqs[at] = make_uint2(~e.y, e.y);   // largest ~j = smallest j
      }
    }
    __syncthreads();
    const int neq = sh.neq;
    uint32_t jmax = 0xffffffffu;                                 // ties taken: index <= jmax
    if (need_eq < neq) {
      if (neq > kSample / 2) {                                   // (more ties than the scratch)
        use_window = false;
      } else {
        int dummy;
        jmax = ~radix_select(sh, eqs, neq, 0u, 0u, 24, need_eq, &dummy, key_x);
      }
    }
    if (use_window) {
      // ---- 3: selected rows -> bitmap -> positions in index order -------------------------
      const int W = (p + 31) / 32;
      uint32_t* bm = reinterpret_cast<uint32_t*>(&sh + 1);
      int* pre = reinterpret_cast<int*>(bm + W);
      for (int w = tid; w < W; w += kThreads) bm[w] = 0u;
      __syncthreads();
      auto taken = [&](uint2 e) {
        const uint32_t key = key_bits(e);
        return key > kth || (key == kth && e.y <= jmax);
      };
      for (int i = tid; i < tot_above; i += kThreads) {
        const uint32_t j = __ldcg(&abuf[i].y);
        atomicOr(bm + (j >> 5), 1u << (j & 31));
      }
      for (int i = tid; i < nc; i += kThreads) {
        const uint2 e = sh.cand[i];
        if (taken(e)) atomicOr(bm + (e.y >> 5), 1u << (e.y & 31));
      }
      __syncthreads();
      const int per = (W + kThreads - 1) / kThreads;
      const int w0 = min(W, tid * per), w1 = min(W, w0 + per);
      int cntw = 0;
      for (int w = w0; w < w1; ++w) cntw += __popc(bm[w]);
      int x = cntw;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(LFPS_FULL, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) sh.wsum[warp] = x;
      __syncthreads();
      int run = x - cntw, total = 0;
      for (int w = 0; w < kWarps; ++w) {
        run += w < warp ? sh.wsum[w] : 0;
        total += sh.wsum[w];
      }
      for (int w = w0; w < w1; ++w) {
        pre[w] = run;
        run += __popc(bm[w]);
      }
      __syncthreads();
      auto emit = [&](uint2 e) {
        const uint32_t j = e.y;
        const int pos = pre[j >> 5] + __popc(bm[j >> 5] & ((1u << (j & 31)) - 1u));
        out_i[pos] = S + (int)j;
        out_z[pos] = __uint_as_float(e.x);
      };
      for (int i = tid; i < tot_above; i += kThreads) emit(__ldcg(&abuf[i]));
      for (int i = tid; i < nc; i += kThreads) {
        const uint2 e = sh.cand[i];
        if (taken(e)) emit(e);
      }
      if (tid == 0) cnt[CNT_C2] = total;
      return;
    }
    __syncthreads();
  }
  // ---- fallback: per-chunk counts, histogram select, ordered emission pass --------------
  uint32_t kth;
  int need_eq;
  const uint2* cand = sh.cand;
  int ncand;
  {
    // ---- fallback: 2048-bin histogram over all keys, then the k-th bin ----------------
    unsigned* hist = sh.samp;                      // 2048 bins
    for (int i = tid; i < kBins; i += kThreads) hist[i] = 0;
    if (tid == 0) sh.ncand = 0;
    __syncthreads();
    for (int j = tid; j < p; j += kThreads) atomicAdd(&hist[key_at(z, j) >> kShift], 1u);
    __syncthreads();
    // thread t owns bins [kBins - 4 t - 4, kBins - 4 t) (descending)
    unsigned loc = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) loc += hist[kBins - 1 - 4 * tid - i];
    unsigned x = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(LFPS_FULL, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sh.wsum[warp] = (int)x;
    __syncthreads();
    unsigned before = 0;
    for (int w = 0; w < warp; ++w) before += (unsigned)sh.wsum[w];
    const unsigned excl = before + x - loc;
    if (excl < (unsigned)k && excl + loc >= (unsigned)k) {
      unsigned cum = excl;
      for (int i = 0; i < 4; ++i) {
        const int bin = kBins - 1 - 4 * tid - i;
        const unsigned hc = hist[bin];
        if (cum + hc >= (unsigned)k) {
          sh.sel_digit = (unsigned)bin;
          sh.sel_want = k - (int)cum;
          break;
        }
        cum += hc;
      }
    }
    __syncthreads();
    const unsigned bstar = sh.sel_digit;
    const int want = sh.sel_want;
    ncand = (int)hist[bstar];
    uint2* store = ncand <= kCand ? sh.cand : reinterpret_cast<uint2*>(c.uw + (size_t)s * c.list_cap);
    __syncthreads();
    int ab = 0;
    for (int j = j0 + lane; j < j1; j += 32) {
      const uint32_t key = key_at(z, j);
      const uint32_t bin = key >> kShift;
      ab += bin > bstar;
      if (bin == bstar) {
        const int at = atomicAdd(&sh.ncand, 1);
        store[at] = make_uint2(key, (uint32_t)j);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) ab += __shfl_xor_sync(LFPS_FULL, ab, o);
    if (lane == 0) sh.above[warp] = ab;
    __syncthreads();
    cand = store;
    kth = radix_select(sh, cand, ncand, bstar << kShift, ~0u << kShift, 16, want, &need_eq, key_x);
    // radix_select's top pass (bits 16..23) covers the remaining 21 bits in 3
    // passes of 8 (bits above 21 already fixed by the prefix)
  }

  // per-warp-chunk counts of window / bin keys above and equal to kth
  for (int i = tid; i < ncand; i += kThreads) {
    const uint2 e = cand[i];
    const int w = (int)e.y / chunk;
    if (e.x > kth) atomicAdd(&sh.gtc[w], 1);
    else if (e.x == kth) atomicAdd(&sh.eqc[w], 1);
  }
  __syncthreads();
  // ---- 3: ordered emission: warp w walks its chunk in index order ---------------------
  int out_at = 0, eq_at = 0;
  for (int w = 0; w < warp; ++w) {
    const int eq = sh.eqc[w];
    out_at += sh.above[w] + sh.gtc[w] + max(0, min(eq, need_eq - eq_at));
    eq_at += eq;
  }
  // the next chunk's float4 is loaded while this one is emitted
  float4 nxt = make_float4(0.f, 0.f, 0.f, 0.f);
  if (vec_ok && j0 + 4 * lane + 3 < j1) nxt = __ldg(reinterpret_cast<const float4*>(z + j0 + 4 * lane));
  for (int base = j0; base < j1; base += 128) {
    // lane owns 4 consecutive keys: j = base + 4 lane + e
    uint32_t keys[4];
    int ntake = 0, neq = 0;
    const float4 cur = nxt;
    if (vec_ok && base + 128 + 4 * lane + 3 < j1)
      nxt = __ldg(reinterpret_cast<const float4*>(z + base + 128 + 4 * lane));
    if (vec_ok && base + 4 * lane + 3 < j1) {
      const float4 v = cur;
      keys[0] = score_key(v.x); keys[1] = score_key(v.y);
      keys[2] = score_key(v.z); keys[3] = score_key(v.w);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int j = base + 4 * lane + e;
        keys[e] = j < j1 ? key_at(z, j) : 0u;
      }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) neq += base + 4 * lane + e < j1 && keys[e] == kth;
    // exclusive warp scans of equal-key counts (index order = lane-major)
    int eqx = neq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(LFPS_FULL, eqx, o);
      if (lane >= o) eqx += y;
    }
    const int eq_total = __shfl_sync(LFPS_FULL, eqx, 31);
    int my_eq = eq_at + eqx - neq;
    bool take[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int j = base + 4 * lane + e;
      const bool eq = j < j1 && keys[e] == kth;
      take[e] = j < j1 && (keys[e] > kth || (eq && my_eq < need_eq));
      my_eq += eq;
      ntake += take[e];
    }
    int tx = ntake;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(LFPS_FULL, tx, o);
      if (lane >= o) tx += y;
    }
    const int take_total = __shfl_sync(LFPS_FULL, tx, 31);
    int pos = out_at + tx - ntake;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (take[e]) {
        const int j = base + 4 * lane + e;
        out_i[pos] = S + j;
        out_z[pos] = z[j];
        ++pos;
      }
    }
    out_at += take_total;
    eq_at += eq_total;
  }
  if (warp == kWarps - 1 && lane == 0) cnt[CNT_C2] = out_at;
}

}  // namespace

cudaError_t launch_topk(const Ctx& c, int /*implicit_base*/, cudaStream_t st) {
  static DeviceOnce once;
  // TopkShared, then the selection bitmap and its word prefixes (list_cap rows)
  const size_t smem = sizeof(TopkShared) + (size_t)(c.list_cap + 31) / 32 * 8;
  cudaError_t e = once.run([&] {
    return cudaFuncSetAttribute(lfps_exact_topk_kernel,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  });
  if (e != cudaSuccess) return e;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  lfps_exact_topk_kernel<<<c.NS, kThreads, smem, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
