// common.cuh -- shared device-side definitions for liblfps_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/lfps_b200.h"

#define LFPS_FULL 0xffffffffu

namespace lfps {

// Table-stage scratch (k_tables.cu, k_probe.cu).
struct TablesWs {
  double* cstat;   // [2 NS][512][4] chunk moments
  int* cidx;       // [2 NS][cap] captured slot indices (logical)
  double* cval;    // [2 NS][cap] captured phys values
  int* ncap;       // [2 NS] capture counts
  int cap;
  double* itemf;   // [2 NS][4] thr0 = tau/scale, thrf = mean/scale, degenerate
  double* bound;   // [2 NS] capture bound for the next step (persists across steps)
  int* fb;         // [2 NS] item took the fallback (C0 bitmap in bits)
  int* fblist;     // [2 NS] queued fallback items
  int* nfb;        // [1]
};

// Flattened per-launch view of dims + state + workspace (passed by value).
struct Ctx {
  // dims
  int B, Hkv, G, Hq, NS, d, n_max, m_cap, ring_cap;
  int words;      // bitmap words per (session, table, kind)
  int list_cap;
  // params
  double r, eps, a, frac, sqrt_d;
  float sqrt_d_f32;
  int s, S, L, bypass_mode, exhaustive, n_off, flags;
  int off[16];
  // state
  const __nv_bfloat16* K;
  const __nv_bfloat16* V;
  __nv_bfloat16* Kw;
  __nv_bfloat16* Vw;
  int* n_ctx;
  double* ver;
  double* sla;
  double* scale;
  int* sla_base;
  long long* clamp_count;
  double* mean_key;
  double* mean_value;
  double* sigma;
  // workspace
  double* rho;
  int* bypass;
  int* err;
  float* out;
  double* thr;
  int* counts;
  uint32_t* bits;
  int* probe_idx;
  float* probe_score;
  int* c2_idx;
  float* c2_score;
  double* scratch;
  TablesWs tb;
};

enum { CNT_C0 = 0, CNT_C1, CNT_PROBE, CNT_DROP, CNT_K, CNT_C2, CNT_CLAMP, CNT_SPARE, CNT_N };

__device__ __forceinline__ const __nv_bfloat16* krow(const Ctx& c, int b, int h, int i) {
  return c.K + (((size_t)b * c.Hkv + h) * c.n_max + i) * c.d;
}
__device__ __forceinline__ const __nv_bfloat16* vrow(const Ctx& c, int b, int h, int i) {
  return c.V + (((size_t)b * c.Hkv + h) * c.n_max + i) * c.d;
}

__device__ __forceinline__ void set_err(const Ctx& c, int s, int code) {
  c.err[1 + s] = code;
  atomicExch(c.err, 1);
}

// ---- host-side launch wrappers (defined in the k_*.cu files) -------------
cudaError_t launch_gate(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st);
cudaError_t launch_tables(const Ctx& c, int m_max, cudaStream_t st);
cudaError_t launch_probe(const Ctx& c, int m_max, cudaStream_t st);
cudaError_t launch_score(const Ctx& c, const __nv_bfloat16* q, int max_list, cudaStream_t st);
cudaError_t launch_topk(const Ctx& c, int implicit_base, cudaStream_t st);
cudaError_t launch_attend(const Ctx& c, const __nv_bfloat16* q, int exact_mode, cudaStream_t st);
cudaError_t launch_update(const Ctx& c, cudaStream_t st);
cudaError_t launch_finish(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st);
cudaError_t launch_append(const Ctx& c, const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                          cudaStream_t st);
cudaError_t launch_commit(const Ctx& c, cudaStream_t st);
cudaError_t launch_boot_tables(const Ctx& c, const float* w, int s_begin, int count, int m0,
                               cudaStream_t st);
cudaError_t launch_boot_stats(const Ctx& c, const __nv_bfloat16* q, int m_max, cudaStream_t st);
cudaError_t launch_exact_score(const Ctx& c, const __nv_bfloat16* q, int m_max, cudaStream_t st);
cudaError_t launch_overlap(const Ctx& c, const int* sel, const int* sel_cnt, const int* ex,
                           const int* ex_cnt, int list_stride, int cnt_stride, double* eta,
                           cudaStream_t st);
cudaError_t launch_clear_err(const Ctx& c, cudaStream_t st);

}  // namespace lfps
