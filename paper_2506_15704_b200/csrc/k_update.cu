// k_update.cu -- tracker update + grow (K6), KV append and commit.
//
// lfps_update_kernel restates ScoreTablePair.update / grow (tables.py:144-220)
// in ring form: u = canonical fp64 softmax of the selected fp32 scores
// (engine.py:184, devmath.softmax_update); |sum u - 1| <= 1e-6 check;
// scale *= r with renormalisation below 1e-120 (vertical [0, m) and slash
// logical [0, m] multiplied by the new scale); slash shift = ring base - 1
// with the new logical slot 0 zeroed and the old top parked at logical m;
// add = (u - 1/(2k)) / scale folded into both tables at C2; negative
// entries clamped to 0 and counted; grow: vertical slot m = 0, slash slot m
// keeps the parked value (zero on bypassed steps, which only grow).
//
// Nothing is committed if any session of the batch raised a data error
// (err[0] != 0): the whole step is atomic (engine.py:8-9).
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads) lfps_update_kernel(Ctx c) {
  __shared__ double red[9];
  __shared__ int clamp_red[kThreads / 32];
  const int s = blockIdx.x, tid = threadIdx.x;
  if (c.err[0] != 0) return;
  const int b = s / c.Hq;
  const int n = c.n_ctx[b];
  const int m = n - c.S;
  const int C = c.ring_cap;
  double* ver = c.ver + (size_t)s * c.m_cap;
  double* sla = c.sla + (size_t)s * C;
  int base = c.sla_base[s];
  if (c.bypass[s]) {
    if (tid == 0) {
      ver[m] = 0.0;
      sla[(base + m) % C] = 0.0;       // no parked carry on a gated step
    }
    return;
  }
  const int k2 = c.counts[(size_t)s * CNT_N + CNT_C2];
  const int* idx = c.c2_idx + (size_t)s * c.list_cap;
  const float* z = c.c2_score + (size_t)s * c.list_cap;
  // max (exact in any order)
  double mx = -INFINITY;
  for (int j = tid; j < k2; j += kThreads) mx = fmax(mx, (double)z[j]);
  for (int o = 16; o >= 1; o >>= 1) mx = fmax(mx, __shfl_xor_sync(LFPS_FULL, mx, o));
  if ((tid & 31) == 0) red[tid >> 5] = mx;
  __syncthreads();
  mx = red[0];
  for (int w = 1; w < kThreads / 32; ++w) mx = fmax(mx, red[w]);
  __syncthreads();
  // canonical sum of exponentials: thread t owns j = t, t + 256, ...
  double acc = 0.0;
  for (int j = tid; j < k2; j += kThreads) acc = cadd(acc, cexp(csub((double)z[j], mx)));
  const double tot = block_fold256(acc, red);
  // sum of the normalised weights (tables.py:161-163)
  acc = 0.0;
  for (int j = tid; j < k2; j += kThreads) acc = cadd(acc, cdiv(cexp(csub((double)z[j], mx)), tot));
  const double wsum = block_fold256(acc, red);
  if (fabs(wsum - 1.0) > 1e-6) {
    if (tid == 0) set_err(c, s, LFPS_ERR_WEIGHT_SUM);
    return;
  }
  // decay with renormalisation (tables.py:167-169, 240-244)
  double sc = cmul(c.scale[s], c.r);
  if (sc < 1e-120) {
    for (int i = tid; i < m; i += kThreads) ver[i] = cmul(ver[i], sc);
    for (int i = tid; i <= m; i += kThreads) {
      const int slot = (base + i) % C;
      sla[slot] = cmul(sla[slot], sc);
    }
    sc = 1.0;
    __syncthreads();
  }
  // slash shift (tables.py:174-177)
  base = (base - 1 + C) % C;
  if (tid == 0) sla[base] = 0.0;
  __syncthreads();
  // residual fold and clamp (tables.py:179-199)
  const double inv = cdiv(1.0, cmul(2.0, (double)k2));
  int clamps = 0;
  for (int j = tid; j < k2; j += kThreads) {
    const double u = cdiv(cexp(csub((double)z[j], mx)), tot);
    const double add = cdiv(csub(u, inv), sc);
    const int li = idx[j] - c.S;
    double v = cadd(ver[li], add);
    if (v < 0.0) { v = 0.0; ++clamps; }
    ver[li] = v;
    const int slot = (base + li) % C;
    double w = cadd(sla[slot], add);
    if (w < 0.0) { w = 0.0; ++clamps; }
    sla[slot] = w;
  }
  for (int o = 16; o >= 1; o >>= 1) clamps += __shfl_xor_sync(LFPS_FULL, clamps, o);
  if ((tid & 31) == 0) clamp_red[tid >> 5] = clamps;
  __syncthreads();
  if (tid == 0) {
    int tc = 0;
    for (int w = 0; w < kThreads / 32; ++w) tc += clamp_red[w];
    c.counts[(size_t)s * CNT_N + CNT_CLAMP] = tc;
    c.clamp_count[s] += tc;
    // grow (tables.py:202-220): the parked slash value at logical m stays
    ver[m] = 0.0;
    c.scale[s] = sc;
    c.sla_base[s] = base;
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
