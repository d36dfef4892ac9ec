// k_gate.cu -- sparsity gate and bypass output (K0).
//
// Restates gate_logits + sparsity_from_logits + bypass_output
// (pkg/src/lfps/gate.py:77-147) and the gate part of decode_step
// (engine.py:127-146) for every session of the batch: one CTA per session,
// fp64 throughout, canonical dot/exp/sum order (canon.cuh).  Sink rows,
// the trailing local rows and the priors are read straight from the bf16 KV
// cache and the fp64 prior buffers.
#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"

namespace lfps {

namespace {

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

// One 128-thread CTA per session: the S + L logit rows are spread over the 4
// warps (each a canonical warp gdot), then warp 0 finishes the gate.  (One
// warp per session walked the rows serially: 2048 warps could not fill the
// GPU and each was a ~70-deep chain of warp folds.)
constexpr int kGateWarps = 4;
constexpr int kMaxRows = 96;     // S <= 31, L <= 64

__global__ void __launch_bounds__(kGateWarps * 32) lfps_gate_kernel(Ctx c, const __nv_bfloat16* q) {
  __shared__ double lg[kMaxRows];   // logits: sinks [0, S), local rows [S, S + L)
  __shared__ double ev[kMaxRows];
  __shared__ double gsh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = c.s_off + blockIdx.x;
  pdl_wait();                                  // the previous step's commit (n_ctx, K rows)
  if (s >= c.NS) return;
  const int b = s / c.Hq, qh = s % c.Hq, h = qh / c.G;
  const int n = c.n_ctx[b];
  const int S = c.S, L = c.L, d = c.d;
  const int m = n - S;
  const int R = S + L;

  double qv[kMaxPerLane];
  const uint16_t* qs = reinterpret_cast<const uint16_t*>(q + (size_t)s * d);
#pragma unroll
  for (int e = 0; e < kMaxPerLane; ++e) {
    const int j = lane + 32 * e;
    qv[e] = (j < d) ? (double)bf2f(qs[j]) : 0.0;
  }
  // logits: sinks [0, S), local rows [n - L, n)  (gate.py:92-94)
  for (int r = warp; r < R; r += kGateWarps) {
    const __nv_bfloat16* row = r < S ? krow(c, b, h, r) : krow(c, b, h, n - L + (r - S));
    const double z = cdiv(row_dot(row, qv, d, lane), c.sqrt_d);
    if (lane == 0) lg[r] = z;
  }
  // global exponent (gate.py:77-81): q.Kbar / sqrt(d) + |q|^2 sigma^2 / 2, by
  // the warp with the fewest rows
  if (warp == (R % kGateWarps)) {
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
    if (lane == 0) gsh = cadd(cdiv(qk, c.sqrt_d), cdiv(cmul(qq, c.sigma[s]), 2.0));
  }
  __syncthreads();
  if (warp != 0) return;
  const double g = gsh;
  bool finite = isfinite(g);
  double sl_max = -INFINITY, ll_max = -INFINITY;
  for (int r = lane; r < R; r += 32) {
    const double z = lg[r];
    finite &= isfinite(z);
    if (r < S) sl_max = fmax(sl_max, z);
    else ll_max = fmax(ll_max, z);
  }
  finite = __all_sync(LFPS_FULL, finite);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    sl_max = fmax(sl_max, __shfl_xor_sync(LFPS_FULL, sl_max, o));
    ll_max = fmax(ll_max, __shfl_xor_sync(LFPS_FULL, ll_max, o));
  }
  if (!finite) {
    if (lane == 0) { set_err(c, s, LFPS_ERR_NONFINITE_LOGITS); c.bypass[s] = 0; c.rho[s] = NAN; }
    return;
  }
  // shared max shift and the three mass terms (gate.py:107-111): the
  // exponentials in parallel, the two sums left to right
  const double shift = fmax(fmax(sl_max, ll_max), g);
  for (int r = lane; r < R; r += 32) ev[r] = cexp(csub(lg[r], shift));
  __syncwarp();
  double rho = 0.0;
  if (lane == 0) {
    double w_s = 0.0, w_l = 0.0;
    for (int i = 0; i < S; ++i) w_s = cadd(w_s, ev[i]);
    for (int i = 0; i < L; ++i) w_l = cadd(w_l, ev[S + i]);
    const double w_g = cmul(cexp(csub(g, shift)), (double)m);
    rho = cdiv(w_s, cadd(cadd(w_s, w_g), w_l));
  }
  rho = __shfl_sync(LFPS_FULL, rho, 0);
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
  const double evs = (lane < S) ? cexp(csub(lg[lane < S ? lane : 0], mx))
                                : (lane == S ? cexp(csub(g, mx)) : 0.0);
  const double tot = warp_fold(evs);
  double w[32];
  for (int i = 0; i <= S; ++i) {
    const double ei = __shfl_sync(LFPS_FULL, evs, i);
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
  return launch_pdl(lfps_gate_kernel, dim3(c.s_cnt), dim3(kGateWarps * 32), 0, st, c, q);
}

}  // namespace lfps
