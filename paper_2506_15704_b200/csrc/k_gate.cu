// k_gate.cu -- sparsity gate and bypass output (K0).
//
// Restates gate_logits + sparsity_from_logits + bypass_output
// (pkg/src/lfps/gate.py:77-147) and the gate part of decode_step
// (engine.py:127-146) for every session of the batch: one warp per session,
// fp64 throughout, canonical dot/exp/sum order (canon.cuh).  Sink rows,
// the trailing local rows and the priors are read straight from the bf16 KV
// cache and the fp64 prior buffers.
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

constexpr int kWarps = 8;
constexpr int kMaxPerLane = 8;  // d <= 256

// Canonical fp64 dot of a bf16 row with the lane-resident query (gdot):
// lane l accumulates j = l, l+32, ... then the warp folds 16..1.
__device__ __forceinline__ double row_dot(const __nv_bfloat16* row, const double* qv, int d,
                                          int lane) {
  const uint16_t* r = reinterpret_cast<const uint16_t*>(row);
  double acc = 0.0;
#pragma unroll
  for (int e = 0; e < kMaxPerLane; ++e) {
    const int j = lane + 32 * e;
    if (j < d) acc = cadd(acc, cmul((double)bf2f(__ldg(r + j)), qv[e]));
  }
  return warp_fold(acc);
}

__global__ void __launch_bounds__(kWarps * 32, 6) lfps_gate_kernel(Ctx c, const __nv_bfloat16* q) {
  const int lane = threadIdx.x & 31;
  const int sidx = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (sidx >= c.s_cnt) return;
  const int s = c.s_off + sidx;
  if (s >= c.NS) return;
  const int b = s / c.Hq, qh = s % c.Hq, h = qh / c.G;
  const int n = c.n_ctx[b];
  const int S = c.S, L = c.L, d = c.d;
  const int m = n - S;
  if (lane == 0) c.counts[(size_t)s * CNT_N + CNT_BLOCKS] = 0;   // summed by k_select.cu

  double qv[kMaxPerLane];
  const uint16_t* qs = reinterpret_cast<const uint16_t*>(q + (size_t)s * d);
#pragma unroll
  for (int e = 0; e < kMaxPerLane; ++e) {
    const int j = lane + 32 * e;
    qv[e] = (j < d) ? (double)bf2f(qs[j]) : 0.0;
  }
  // logits: sinks [0, S), local rows [n - L, n)  (gate.py:92-94)
  double sl_max = -INFINITY, ll_max = -INFINITY;
  double sl[32];           // S <= 31
  double ll[64];           // L <= 64
  bool finite = true;
  for (int i = 0; i < S; ++i) {
    sl[i] = cdiv(row_dot(krow(c, b, h, i), qv, d, lane), c.sqrt_d);
    finite &= isfinite(sl[i]);
    sl_max = fmax(sl_max, sl[i]);
  }
  for (int i = 0; i < L; ++i) {
    ll[i] = cdiv(row_dot(krow(c, b, h, n - L + i), qv, d, lane), c.sqrt_d);
    finite &= isfinite(ll[i]);
    ll_max = fmax(ll_max, ll[i]);
  }
  // global exponent (gate.py:77-81): q.Kbar / sqrt(d) + |q|^2 sigma^2 / 2
  const double* kbar = c.mean_key + ((size_t)b * c.Hkv + h) * d;
  double qk = 0.0, qq = 0.0;
#pragma unroll
  for (int e = 0; e < kMaxPerLane; ++e) {
    const int j = lane + 32 * e;
    if (j < d) {
      qk = cadd(qk, cmul(qv[e], kbar[j]));
      qq = cadd(qq, cmul(qv[e], qv[e]));
    }
  }
  qk = warp_fold(qk);
  qq = warp_fold(qq);
  const double g = cadd(cdiv(qk, c.sqrt_d), cdiv(cmul(qq, c.sigma[s]), 2.0));
  finite &= isfinite(g);
  if (!finite) {
    if (lane == 0) { set_err(c, s, LFPS_ERR_NONFINITE_LOGITS); c.bypass[s] = 0; c.rho[s] = NAN; }
    return;
  }
  // shared max shift and the three mass terms (gate.py:107-111)
  const double shift = fmax(fmax(sl_max, ll_max), g);
  double w_s = 0.0, w_l = 0.0;
  for (int i = 0; i < S; ++i) w_s = cadd(w_s, cexp(csub(sl[i], shift)));
  for (int i = 0; i < L; ++i) w_l = cadd(w_l, cexp(csub(ll[i], shift)));
  const double w_g = cmul(cexp(csub(g, shift)), (double)m);
  const double rho = cdiv(w_s, cadd(cadd(w_s, w_g), w_l));
  if (!isfinite(rho)) {
    if (lane == 0) { set_err(c, s, LFPS_ERR_NONFINITE_RHO); c.bypass[s] = 0; c.rho[s] = rho; }
    return;
  }
  const int gated = rho > c.eps;
  if (lane == 0) { c.rho[s] = rho; c.bypass[s] = gated; }
  if (!gated) return;

  // bypass output (gate.py:131-147)
  float* out = c.out + (size_t)s * d;
  const double* vbar = c.mean_value + ((size_t)b * c.Hkv + h) * d;
  if (c.bypass_mode == 1) {
    for (int j = lane; j < d; j += 32) out[j] = (float)vbar[j];
    return;
  }
  // softmax over [sink logits..., g]: max, cexp, 256-thread canonical sum
  // (for <= 32 terms the warp fold is the block fold), divide.
  double mx = fmax(sl_max, g);
  const double ev = (lane < S) ? cexp(csub(sl[lane < S ? lane : 0], mx))
                               : (lane == S ? cexp(csub(g, mx)) : 0.0);
  const double tot = warp_fold(ev);
  double w[32];
  for (int i = 0; i <= S; ++i) {
    const double ei = __shfl_sync(LFPS_FULL, ev, i);
    w[i] = cdiv(ei, tot);
  }
  for (int j = lane; j < d; j += 32) {
    double acc = 0.0;
    for (int i = 0; i < S; ++i) {
      const uint16_t* vr = reinterpret_cast<const uint16_t*>(vrow(c, b, h, i));
      acc = cadd(acc, cmul(w[i], (double)bf2f(vr[j])));
    }
    acc = cadd(acc, cmul(w[S], vbar[j]));
    out[j] = (float)acc;
  }
}

}  // namespace

cudaError_t launch_gate(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  const int blocks = (c.s_cnt + kWarps - 1) / kWarps;
  lfps_gate_kernel<<<blocks, kWarps * 32, 0, st>>>(c, q);
  return cudaGetLastError();
}

}  // namespace lfps
