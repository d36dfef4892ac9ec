// k_bootstrap.cu -- prefill bootstrap on the device (next-row N1).
//
// lfps_boot_tables_kernel  : Eq. 4 seeding (init_tables, tables.py:247-281); rows
//                       accumulated oldest first, exactly numpy's axis-0 order,
//                       so the seeded tables equal the reference's bit for bit.
// lfps_boot_rowsum_kernel  : each prefill weight row sums to 1 within 1e-4
//                       (prefill_bootstrap, engine.py:84-86).
// lfps_boot_mean_kernel    : K-bar / V-bar over the non-sink rows, rows summed in
//                       order (numpy's keys_ns.mean(axis=0), gate.py:71-72).
// lfps_boot_logit_kernel + lfps_boot_sigma_kernel : sigma_hat^2 = var(logits) / |q|^2
//                       with canonical fp64 dots and chunked sums
//                       (gate.py:61-67, devmath DevArith.head_sigma).
#include "common.cuh"
#include "canon.cuh"

namespace lfps {

namespace {

__global__ void lfps_boot_tables_kernel(Ctx c, const float* w, int s_begin, int m0) {
  const int sl = blockIdx.y;
  const int s = s_begin + sl;
  const int sp = c.s;
  const float* ws = w + (size_t)sl * sp * m0;
  double* ver = ver_row(c, s);
  double* sla = sla_row(c, s);
  const int base0 = c.sla_home - m0;    // the slash window ends at the home slot
  const double coeff = cdiv(1.0, cmul(cmul(2.0, (double)sp), csub(1.0, c.r)));
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < c.sla_cap; i += gridDim.x * blockDim.x) {
    double col = 0.0, diag = 0.0;
    if (i < m0) {
      for (int r = 0; r < sp; ++r) {
        col = cadd(col, (double)ws[(size_t)r * m0 + i]);
        const int lag = sp - 1 - r;
        if (lag <= i) diag = cadd(diag, (double)ws[(size_t)r * m0 + i - lag]);
      }
      col = cmul(col, coeff);
      diag = cmul(diag, coeff);
    }
    if (i < c.m_cap) ver[i] = col;
    // slot base0 + i holds logical i; zero everywhere else
    const int li = i - base0;
    if (li < 0 || li >= m0) sla[i] = 0.0;
    if (i < m0) sla[base0 + i] = diag;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.scale[s] = 1.0;
    c.sla_base[s] = base0;
    c.clamp_count[s] = 0;
    c.bw.valid[s] = 0;                  // the next step rebuilds every block summary
  }
}

__global__ void lfps_boot_rowsum_kernel(Ctx c, const float* w, int s_begin, int m0) {
  __shared__ double red[32];
  const int sl = blockIdx.x, r = blockIdx.y;
  const float* row = w + ((size_t)sl * c.s + r) * m0;
  double acc = 0.0;
  for (int i = threadIdx.x; i < m0; i += blockDim.x) acc += (double)row[i];
  for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(LFPS_FULL, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    if (fabs(t - 1.0) > 1e-4) set_err(c, s_begin + sl, LFPS_ERR_PREFILL_SUM);
  }
}

// one CTA per unit, one thread per (matrix, column): sequential row sums
__global__ void lfps_boot_mean_kernel(Ctx c, int u0) {
  const int u = u0 + blockIdx.x;
  const int b = u / c.Hkv, h = u % c.Hkv;
  const int n = c.n_ctx[b];
  const int S = c.S, d = c.d;
  const int t = threadIdx.x;
  if (t >= 2 * d) return;
  const int j = t % d;
  const uint16_t* src = reinterpret_cast<const uint16_t*>(t < d ? c.K : c.V) + j;
  const RowMap rm(c, b, h);
  double acc = 0.0;
  int i = S;
  for (; i + 4 <= n; i += 4) {
    const float a0 = bf2f(src[(size_t)rm(i) * d]);
    const float a1 = bf2f(src[(size_t)rm(i + 1) * d]);
    const float a2 = bf2f(src[(size_t)rm(i + 2) * d]);
    const float a3 = bf2f(src[(size_t)rm(i + 3) * d]);
    acc = cadd(acc, (double)a0);
    acc = cadd(acc, (double)a1);
    acc = cadd(acc, (double)a2);
    acc = cadd(acc, (double)a3);
  }
  for (; i < n; ++i) acc = cadd(acc, (double)bf2f(src[(size_t)rm(i) * d]));
  const double mean = cdiv(acc, (double)(n - S));
  (t < d ? c.mean_key : c.mean_value)[(size_t)u * d + j] = mean;
}

// logits of every non-sink row for every session of a unit -> scratch
__global__ void lfps_boot_logit_kernel(Ctx c, const __nv_bfloat16* q, int u0) {
  const int u = u0 + blockIdx.y;
  const int b = u / c.Hkv, h = u % c.Hkv;
  const int n = c.n_ctx[b];
  const int S = c.S, d = c.d;
  const int lane = threadIdx.x & 31;
  const int warps = blockDim.x >> 5;
  for (int g = 0; g < c.G; ++g) {
    const int s = b * c.Hq + h * c.G + g;
    double qv[8];
    const uint16_t* qs = reinterpret_cast<const uint16_t*>(q + (size_t)s * d);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = lane + 32 * e;
      qv[e] = j < d ? (double)bf2f(qs[j]) : 0.0;
    }
    for (int i = S + blockIdx.x * warps + (threadIdx.x >> 5); i < n; i += gridDim.x * warps) {
      const uint16_t* r = reinterpret_cast<const uint16_t*>(krow(c, b, h, i));
      double acc = 0.0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = lane + 32 * e;
        if (j < d) acc = cadd(acc, cmul((double)bf2f(r[j]), qv[e]));
      }
      acc = warp_fold(acc);
      if (lane == 0) c.scratch[(size_t)s * c.list_cap + (i - S)] = cdiv(acc, c.sqrt_d);
    }
  }
}

// canonical chunked sum (devmath.table_sum) of x[0, cnt) by one CTA of
// 256 threads; partials: smem scratch of >= ceil(cnt/512) rounded to pow2
template <bool CENTRED>
__device__ double block_table_sum(const double* x, int cnt, double mu, double* parts, int n2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = (cnt + 511) / 512;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) parts[i] = 0.0;
  __syncthreads();
  for (int ch = warp; ch < nch; ch += blockDim.x >> 5) {
    double v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int i = ch * 512 + e * 32 + lane;
      v[e] = 0.0;
      if (i < cnt) {
        double t = x[i];
        if (CENTRED) { t = csub(t, mu); t = cmul(t, t); }
        v[e] = t;
      }
    }
    double acc = warp_fold(lane_tree16(v));
    if (lane == 0) parts[ch] = acc;
  }
  __syncthreads();
  double tot = 0.0;
  if (warp == 0) tot = warp_pairwise_tree(parts, n2, lane);
  __syncthreads();
  if (threadIdx.x == 0) parts[0] = tot;
  __syncthreads();
  tot = parts[0];
  __syncthreads();
  return tot;
}

__global__ void lfps_boot_sigma_kernel(Ctx c, const __nv_bfloat16* q, int n2, int s0) {
  extern __shared__ double parts[];
  const int s = s0 + blockIdx.x;
  const int b = s / c.Hq;
  const int cnt = c.n_ctx[b] - c.S;
  const double* x = c.scratch + (size_t)s * c.list_cap;
  const double tot = block_table_sum<false>(x, cnt, 0.0, parts, n2);
  const double mu = cdiv(tot, (double)cnt);
  const double ss = block_table_sum<true>(x, cnt, mu, parts, n2);
  const double var = cdiv(ss, (double)cnt);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const uint16_t* qs = reinterpret_cast<const uint16_t*>(q + (size_t)s * c.d);
    double acc = 0.0;
    for (int e = 0; e < 8; ++e) {
      const int j = lane + 32 * e;
      if (j < c.d) {
        const double v = (double)bf2f(qs[j]);
        acc = cadd(acc, cmul(v, v));
      }
    }
    const double qq = warp_fold(acc);
    if (lane == 0) {
      if (qq == 0.0) set_err(c, s, LFPS_ERR_ZERO_QUERY);
      c.sigma[s] = cdiv(var, qq);
    }
  }
}

}  // namespace

cudaError_t launch_boot_tables(const Ctx& c, const float* w, int s_begin, int count, int m0,
                               cudaStream_t st) {
  const int blocks = (c.sla_cap + 255) / 256;
  lfps_boot_tables_kernel<<<dim3(blocks < 1024 ? blocks : 1024, count), 256, 0, st>>>(c, w, s_begin, m0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  lfps_boot_rowsum_kernel<<<dim3(count, c.s), 256, 0, st>>>(c, w, s_begin, m0);
  return cudaGetLastError();
}

cudaError_t launch_boot_stats(const Ctx& c, const __nv_bfloat16* q, int m_max, int b0, int nb,
                              cudaStream_t st) {
  const int units = nb * c.Hkv, u0 = b0 * c.Hkv;
  lfps_boot_mean_kernel<<<units, 2 * c.d, 0, st>>>(c, u0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int per_unit = (148 * 8 + units - 1) / units;
  if (per_unit > 256) per_unit = 256;
  lfps_boot_logit_kernel<<<dim3(per_unit, units), 256, 0, st>>>(c, q, u0);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int nch = (m_max + 511) / 512;
  int n2 = 1;
  while (n2 < nch) n2 <<= 1;
  if (n2 < 32) n2 = 32;
  lfps_boot_sigma_kernel<<<nb * c.Hq, 256, n2 * sizeof(double), st>>>(c, q, n2, b0 * c.Hq);
  return cudaGetLastError();
}

}  // namespace lfps
