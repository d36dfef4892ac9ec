// k_update.cu -- commit of a decode step in ONE kernel: tracker update +
// grow (K6), KV append and the context count.
//
// lfps_update_kernel restates ScoreTablePair.update / grow (tables.py:144-220)
// on the linear slash window: u = canonical fp64 softmax of the selected
// fp32 scores (engine.py:184, devmath.softmax_update) with the C2 max from
// the finish kernel, checked (|sum u - 1| <= 1e-6); scale *= r with
// renormalisation below 1e-120 (vertical [0, m) and
// slash logical [0, m] multiplied by the new scale); slash shift = base - 1
// with the new logical slot 0 zeroed and the old top parked at logical m;
// add = (u - 1/(2k)) / scale folded into both tables at C2; negative
// entries clamped to 0 and counted; grow: vertical slot m = 0, slash slot m
// keeps the parked value (a gated step only grows, with a zero slash slot).
// Every block whose slots changed is marked dirty for k_select.cu; a
// renormalisation invalidates all of the session's block summaries.
//
// Nothing is committed if any session of the batch raised a data error
// (err[0] == this call's stamp): the whole step is atomic (engine.py:8-9).
#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxDirtyWords = 32;
constexpr int kMaxE = 8;                 // update weights cached per thread (|C2| <= 2048)
#ifndef LFPS_UPDATE_SPEC
#define LFPS_UPDATE_SPEC 4
#endif
constexpr int kSpec = LFPS_UPDATE_SPEC;  // C2 entries per thread fetched with the prologue

// canonical 256-wide block sum (devmath.block_sum); all threads get it
__device__ __forceinline__ double block_sum256(double acc, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  acc = warp_fold(acc);
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    double v = lane < 8 ? red[lane] : 0.0;
#pragma unroll
    for (int h = 4; h >= 1; h >>= 1) v = cadd(v, __shfl_xor_sync(LFPS_FULL, v, h));
    if (lane == 0) red[8] = v;
  }
  __syncthreads();
  const double out = red[8];
  __syncthreads();
  return out;
}
#ifndef LFPS_UPDATE_UNROLL
#define LFPS_UPDATE_UNROLL 2
#endif
constexpr int kUnroll = LFPS_UPDATE_UNROLL;   // C2 entries per thread in flight
#ifndef LFPS_UPDATE_CTAS
#define LFPS_UPDATE_CTAS 6
#endif

__device__ __forceinline__ void mark(uint32_t (*dmark)[kMaxDirtyWords], int t, int blk) {
  atomicOr(&dmark[t][blk >> 5], 1u << (blk & 31));
}

// One CTA per session: the session's table update, the unit's KV append (by
// the unit's first q-head), and -- in the last CTA to finish -- the context
// count of every request (store.py:64-77 append, then engine.py:188-191).
__global__ void __launch_bounds__(kThreads, LFPS_UPDATE_CTAS) lfps_update_kernel(Ctx c, const __nv_bfloat16* k_new,
                                                               const __nv_bfloat16* v_new) {
  __shared__ uint32_t dmark[2][kMaxDirtyWords];
  __shared__ int clamp_red[kThreads / 32];
  __shared__ double red[16];
  const int s = blockIdx.x, tid = threadIdx.x;
  const int b = s / c.Hq, qh = s % c.Hq;
  pdl_wait();                                 // the finish kernel's lists and scores
  // independent prologue loads, issued together
  const int ep = call_stamp(c);
  const int failed = c.err[0] == ep;
  const int n = c.n_ctx[b];
  int base = c.sla_base[s];
  const int byp = c.bypass[s];
  const double sc0 = c.scale[s];
  const int k2 = c.counts[(size_t)s * CNT_N + CNT_C2];
  // the first kSpec C2 entries of this thread, fetched with the prologue
  // (before k2 is known; entries at or beyond k2 are ignored below)
  const int* idx = c.c2_idx + (size_t)s * c.list_cap;
  const float* c2z = c.c2_score + (size_t)s * c.list_cap;
  const double mx = c.bw.wstat[2 * (size_t)s];
  float zs[kSpec];
  int is[kSpec];
#pragma unroll
  for (int i = 0; i < kSpec; ++i) {
    const int j = tid + i * kThreads;
    zs[i] = j < c.list_cap ? c2z[j] : 0.0f;
    is[i] = j < c.list_cap ? idx[j] : 0;
  }
  if (failed) return;                         // a failed step commits nothing
  const int m = n - c.S;
  double* ver = ver_row(c, s);
  double* sla = sla_row(c, s);
  const int dw = c.bw.dwords;
  uint32_t* dirty = c.bw.dirty + (size_t)(2 * s) * dw;
  // KV append of the unit's new row at position n (one session per unit)
  if (qh % c.G == 0) {
    const int u = b * c.Hkv + qh / c.G;
    const size_t row = (size_t)RowMap(c, b, qh / c.G)(n) * c.d;
    __nv_bfloat16* kd = c.Kw + row;
    __nv_bfloat16* vd = c.Vw + row;
    for (int t = tid; t < c.d; t += kThreads) {
      kd[t] = k_new[(size_t)u * c.d + t];
      vd[t] = v_new[(size_t)u * c.d + t];
    }
  }
  if (byp) {
    if (tid == 0) {                     // grow only (engine.py:133-137)
      ver[m] = 0.0;
      sla[base + m] = 0.0;              // no parked carry on a gated step
      const int bv = m / kBlk, bs = (base + m) / kBlk;
      dirty[bv >> 5] |= 1u << (bv & 31);
      dirty[dw + (bs >> 5)] |= 1u << (bs & 31);
    }
  } else {
    for (int i = tid; i < 2 * kMaxDirtyWords; i += kThreads) (&dmark[0][0])[i] = 0u;
    // the slot below the window becomes the new logical slot 0 (it is outside
    // the window until then, so zeroing it early commits nothing)
    if (tid == 0) sla[base - 1] = 0.0;
    // update weights u = canonical fp64 softmax of the C2 scores
    // (devmath.softmax_update, engine.py:184) with the C2 max from the finish
    // kernel; thread t owns entries t + 256 i, exactly the entries it folds
    // below.  The |sum u - 1| <= 1e-6 check (tables.py:161-163) cannot fail
    // for finite scores (the max term is exactly 1, every u rounds once); if it
    // ever did, this session alone would skip its update and only grow
    // (err[0] = -stamp).
    double e[kMaxE];
    int lix[kMaxE];                       // logical C2 index of entry i (-1: none)
    float zi[kMaxE];
#pragma unroll
    for (int i = 0; i < kMaxE; ++i) {     // one round trip for scores and indices
      const int j = tid + i * kThreads;
      if (i < kSpec) {
        zi[i] = j < k2 ? zs[i] : 0.0f;
        lix[i] = j < k2 ? is[i] - c.S : -1;
      } else {
        zi[i] = j < k2 ? c2z[j] : 0.0f;
        lix[i] = j < k2 ? idx[j] - c.S : -1;
      }
    }
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxE; ++i) {
      const int j = tid + i * kThreads;
      e[i] = j < k2 ? cexp(csub((double)zi[i], mx)) : 0.0;
      if (j < k2) acc = cadd(acc, e[i]);
    }
    for (int j = tid + kMaxE * kThreads; j < k2; j += kThreads) acc = cadd(acc, cexp(csub((double)c2z[j], mx)));
    const double tot = block_sum256(acc, red);
    acc = 0.0;
#pragma unroll
    for (int i = 0; i < kMaxE; ++i) {
      const int j = tid + i * kThreads;
      if (j < k2) {
        e[i] = cdiv(e[i], tot);
        acc = cadd(acc, e[i]);
      }
    }
    for (int j = tid + kMaxE * kThreads; j < k2; j += kThreads)
      acc = cadd(acc, cdiv(cexp(csub((double)c2z[j], mx)), tot));
    const double wsum = block_sum256(acc, red);
    const bool wok = fabs(wsum - 1.0) <= 1e-6;        // block-uniform
    if (!wok && tid == 0) {                  // reported, but not as a failed step:
      c.err[1 + s] = err_code(c, LFPS_ERR_WEIGHT_SUM);   // the other sessions commit
      atomicExch(c.err, -ep);
      // the unit's row is still appended, so this session's tables grow like a
      // gated step's (no update) and stay in step with the KV store
      ver[m] = 0.0;
      sla[base + m] = 0.0;
      const int bv = m / kBlk, bs = (base + m) / kBlk;
      dirty[bv >> 5] |= 1u << (bv & 31);
      dirty[dw + (bs >> 5)] |= 1u << (bs & 31);
    }
    if (wok) {
      // decay with renormalisation (tables.py:167-169, 240-244)
      double sc = cmul(sc0, c.r);
      bool renorm = false;
      if (sc < 1e-120) {
        for (int i = tid; i < m; i += kThreads) ver[i] = cmul(ver[i], sc);
        for (int i = tid; i <= m; i += kThreads) sla[base + i] = cmul(sla[base + i], sc);
        sc = 1.0;
        renorm = true;
      }
      // slash shift (tables.py:174-177): the new logical slot 0 (base - 1) was
      // zeroed at the top of this branch; the weight sums' barriers order it
      // before the fold
      base -= 1;
      if (renorm) __syncthreads();                     // block-uniform
      // residual fold and clamp (tables.py:179-199), kUnroll entries in flight
      const double inv = cdiv(1.0, cmul(2.0, (double)k2));
      int clamps = 0;
      // entries j = tid + 256 i, i = i0 .. i0 + kUnroll - 1 (weights of i < kMaxE
      // cached in registers: the i loop is unrolled so e[] stays in registers)
      auto fold = [&](const int* li, const double* u) {
        double v0[kUnroll], w0[kUnroll];
#pragma unroll
        for (int r = 0; r < kUnroll; ++r) {
          v0[r] = li[r] >= 0 ? ver[li[r]] : 0.0;
          w0[r] = li[r] >= 0 ? sla[base + li[r]] : 0.0;
        }
#pragma unroll
        for (int r = 0; r < kUnroll; ++r) {
          if (li[r] < 0) continue;
          const double add = cdiv(csub(u[r], inv), sc);
          double v = cadd(v0[r], add);
          if (v < 0.0) { v = 0.0; ++clamps; }
          ver[li[r]] = v;
          const int slot = base + li[r];
          double w = cadd(w0[r], add);
          if (w < 0.0) { w = 0.0; ++clamps; }
          sla[slot] = w;
          mark(dmark, 0, li[r] / kBlk);
          mark(dmark, 1, slot / kBlk);
        }
      };
#pragma unroll
      for (int i0 = 0; i0 < kMaxE; i0 += kUnroll) {
        if (tid + i0 * kThreads >= k2) break;
        double u[kUnroll];
        int li[kUnroll];
#pragma unroll
        for (int r = 0; r < kUnroll; ++r) {
          u[r] = e[i0 + r];
          li[r] = lix[i0 + r];
        }
        fold(li, u);
      }
      for (int i0 = kMaxE; tid + i0 * kThreads < k2; i0 += kUnroll) {
        double u[kUnroll];
        int li[kUnroll];
#pragma unroll
        for (int r = 0; r < kUnroll; ++r) {
          const int j = tid + (i0 + r) * kThreads;
          u[r] = j < k2 ? cdiv(cexp(csub((double)c2z[j], mx)), tot) : 0.0;
          li[r] = j < k2 ? idx[j] - c.S : -1;
        }
        fold(li, u);
      }
      for (int o = 16; o >= 1; o >>= 1) clamps += __shfl_xor_sync(LFPS_FULL, clamps, o);
      if ((tid & 31) == 0) clamp_red[tid >> 5] = clamps;
      if (tid == 0) {
        // grow (tables.py:202-220): vertical slot m, slash slot base (new logical 0)
        mark(dmark, 0, m / kBlk);
        mark(dmark, 1, base / kBlk);
      }
      __syncthreads();
      if (tid < 2 * dw) {
        const int t = tid / dw, w = tid % dw;
        const uint32_t mk = dmark[t][w];
        if (mk) dirty[t * dw + w] |= mk;
      }
      if (tid == 0) {
        int tc = 0;
        for (int w = 0; w < kThreads / 32; ++w) tc += clamp_red[w];
        c.counts[(size_t)s * CNT_N + CNT_CLAMP] = tc;
        c.clamp_count[s] += tc;
        ver[m] = 0.0;                       // the parked slash value at logical m stays
        c.scale[s] = sc;
        c.sla_base[s] = base;
        if (renorm) c.bw.valid[s] = 0;
      }
    }
  }
  // the last CTA publishes the new context lengths (every n_ctx reader is done)
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(c.done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence();
      for (int r = 0; r < c.B; ++r) c.n_ctx[r] += 1;
      *c.done = 0u;
      // err[0] after a step: 0 = committed (a stale stamp of an earlier failed
      // call is dropped here), this call's stamp = failed
      const int e0 = atomicAdd(c.err, 0);
      if (e0 != ep && e0 != -ep) c.err[0] = 0;
    }
  }
  pdl_trigger();
}

// first node of a CUDA-graph decode step: the step's call stamp, drawn in
// device memory from [2^26, 2^27 - 2) (host-drawn stamps are below 2^26)
__global__ void lfps_step_begin_kernel(int* stamp) {
  int e = *stamp + 1;
  if (e < (1 << 26) || e >= (1 << 27) - 2) e = 1 << 26;
  *stamp = e;
}

__global__ void lfps_clear_err_kernel(Ctx c) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i <= c.NS; i += blockDim.x * gridDim.x)
    c.err[i] = 0;
}

}  // namespace

cudaError_t launch_update(const Ctx& c, const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                          cudaStream_t st) {
  return launch_pdl(lfps_update_kernel, dim3(c.NS), dim3(kThreads), 0, st, c, k_new, v_new);
}

cudaError_t launch_step_begin(const Ctx& c, cudaStream_t st) {
  lfps_step_begin_kernel<<<1, 1, 0, st>>>(const_cast<int*>(c.stamp));
  return cudaGetLastError();
}

cudaError_t launch_clear_err(const Ctx& c, cudaStream_t st) {
  lfps_clear_err_kernel<<<(c.NS + 256) / 256, 256, 0, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
