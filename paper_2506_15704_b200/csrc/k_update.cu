// k_update.cu -- commit of a decode step: tracker update + grow (K6), KV
// append and the context count.
//
// lfps_update_kernel restates ScoreTablePair.update / grow (tables.py:144-220)
// on the linear slash window: u = canonical fp64 softmax of the selected
// fp32 scores (engine.py:184, devmath.softmax_update), computed and checked
// (|sum u - 1| <= 1e-6) by the finish kernel, read from uw; scale *= r with renormalisation below 1e-120 (vertical [0, m) and
// slash logical [0, m] multiplied by the new scale); slash shift = base - 1
// with the new logical slot 0 zeroed and the old top parked at logical m;
// add = (u - 1/(2k)) / scale folded into both tables at C2; negative
// entries clamped to 0 and counted; grow: vertical slot m = 0, slash slot m
// keeps the parked value (a gated step only grows, with a zero slash slot).
// Every block whose slots changed is marked dirty for k_select.cu; a
// renormalisation invalidates all of the session's block summaries.
//
// Nothing is committed if any session of the batch raised a data error
// (err[0] != 0): the whole step is atomic (engine.py:8-9).
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxDirtyWords = 32;

__global__ void __launch_bounds__(kThreads) lfps_update_kernel(Ctx c) {
  __shared__ uint32_t dmark[2][kMaxDirtyWords];
  __shared__ int clamp_red[kThreads / 32];
  const int s = blockIdx.x, tid = threadIdx.x;
  if (c.err[0] != 0) return;
  const int b = s / c.Hq;
  const int n = c.n_ctx[b];
  const int m = n - c.S;
  double* ver = ver_row(c, s);
  double* sla = sla_row(c, s);
  int base = c.sla_base[s];
  const int dw = c.bw.dwords;
  uint32_t* dirty = c.bw.dirty + (size_t)(2 * s) * dw;
  if (c.bypass[s]) {
    if (tid == 0) {                     // grow only (engine.py:133-137)
      ver[m] = 0.0;
      sla[base + m] = 0.0;              // no parked carry on a gated step
      const int bv = m / kBlk, bs = (base + m) / kBlk;
      dirty[bv >> 5] |= 1u << (bv & 31);
      dirty[dw + (bs >> 5)] |= 1u << (bs & 31);
    }
    return;
  }
  for (int i = tid; i < 2 * kMaxDirtyWords; i += kThreads) (&dmark[0][0])[i] = 0u;
  const int k2 = c.counts[(size_t)s * CNT_N + CNT_C2];
  const int* idx = c.c2_idx + (size_t)s * c.list_cap;
  const double* uw = c.uw + (size_t)s * c.list_cap;
  // decay with renormalisation (tables.py:167-169, 240-244)
  double sc = cmul(c.scale[s], c.r);
  bool renorm = false;
  if (sc < 1e-120) {
    for (int i = tid; i < m; i += kThreads) ver[i] = cmul(ver[i], sc);
    for (int i = tid; i <= m; i += kThreads) sla[base + i] = cmul(sla[base + i], sc);
    sc = 1.0;
    renorm = true;
  }
  // slash shift (tables.py:174-177)
  base -= 1;
  __syncthreads();
  if (tid == 0) sla[base] = 0.0;
  __syncthreads();
  // residual fold and clamp (tables.py:179-199)
  const double inv = cdiv(1.0, cmul(2.0, (double)k2));
  int clamps = 0;
  for (int j = tid; j < k2; j += kThreads) {
    const double add = cdiv(csub(uw[j], inv), sc);
    const int li = idx[j] - c.S;
    double v = cadd(ver[li], add);
    if (v < 0.0) { v = 0.0; ++clamps; }
    ver[li] = v;
    const int slot = base + li;
    double w = cadd(sla[slot], add);
    if (w < 0.0) { w = 0.0; ++clamps; }
    sla[slot] = w;
    const int bv = li / kBlk, bs = slot / kBlk;
    atomicOr(&dmark[0][bv >> 5], 1u << (bv & 31));
    atomicOr(&dmark[1][bs >> 5], 1u << (bs & 31));
  }
  for (int o = 16; o >= 1; o >>= 1) clamps += __shfl_xor_sync(LFPS_FULL, clamps, o);
  if ((tid & 31) == 0) clamp_red[tid >> 5] = clamps;
  if (tid == 0) {
    // grow (tables.py:202-220): vertical slot m, slash slot base (new logical 0)
    const int bv = m / kBlk, bs = base / kBlk;
    atomicOr(&dmark[0][bv >> 5], 1u << (bv & 31));
    atomicOr(&dmark[1][bs >> 5], 1u << (bs & 31));
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

// K/V append of the step's new rows at position n (store.py:64-77).
__global__ void lfps_append_kernel(Ctx c, const __nv_bfloat16* k_new, const __nv_bfloat16* v_new) {
  if (c.err[0] != 0) return;
  const int u = blockIdx.x;
  const int b = u / c.Hkv, h = u % c.Hkv;
  const int n = c.n_ctx[b];
  __nv_bfloat16* kd = c.Kw + (((size_t)b * c.Hkv + h) * c.n_max + n) * c.d;
  __nv_bfloat16* vd = c.Vw + (((size_t)b * c.Hkv + h) * c.n_max + n) * c.d;
  for (int t = threadIdx.x; t < c.d; t += blockDim.x) {
    kd[t] = k_new[(size_t)u * c.d + t];
    vd[t] = v_new[(size_t)u * c.d + t];
  }
}

// Publish the new context length after every reader of n is done.
__global__ void lfps_commit_kernel(Ctx c) {
  if (c.err[0] != 0) return;
  for (int b = threadIdx.x; b < c.B; b += blockDim.x) c.n_ctx[b] += 1;
}

__global__ void lfps_clear_err_kernel(Ctx c) {
  for (int i = threadIdx.x + blockIdx.x * blockDim.x; i <= c.NS; i += blockDim.x * gridDim.x)
    c.err[i] = 0;
}

}  // namespace

cudaError_t launch_update(const Ctx& c, cudaStream_t st) {
  lfps_update_kernel<<<c.NS, kThreads, 0, st>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_append(const Ctx& c, const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                          cudaStream_t st) {
  lfps_append_kernel<<<c.B * c.Hkv, 128, 0, st>>>(c, k_new, v_new);
  return cudaGetLastError();
}

cudaError_t launch_commit(const Ctx& c, cudaStream_t st) {
  lfps_commit_kernel<<<1, 256, 0, st>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_clear_err(const Ctx& c, cudaStream_t st) {
  lfps_clear_err_kernel<<<(c.NS + 256) / 256, 256, 0, st>>>(c);
  return cudaGetLastError();
}

}  // namespace lfps
