// common.cuh -- shared device-side definitions for liblfps_b200 (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/lfps_b200.h"

#define LFPS_FULL 0xffffffffu

namespace lfps {

// Persistent block summaries of the tracker tables (k_select.cu, k_update.cu).
// item = 2 s + table; block b = table slots [512 b, 512 b + 512) within the
// item's window (vertical [0, m), slash [base, base + m)).
constexpr int kBlk = 512;
struct BlockWs {
  double* bsum;     // [2 NS][nblk][4] segment mean, M2, M3, M4
  double* bmax;     // [2 NS][nblk] segment max phys value
  uint32_t* dirty;  // [2 NS][dwords] blocks to rebuild at the next step
  int* valid;       // [NS] 0: rebuild every block of the session
  double* wstat;    // [NS][2] update-softmax max and normaliser (finish -> update)
  int nblk;
  int dwords;
};

// Flattened per-launch view of dims + state + workspace (passed by value).
struct Ctx {
  // dims
  int B, Hkv, G, Hq, NS, d, n_max, m_cap, sla_cap, sla_home;
  int words;      // bitmap words per (session, table, kind)
  int list_cap;
  // params
  double r, eps, a, frac, sqrt_d;
  float sqrt_d_f32;
  int s, S, L, bypass_mode, exhaustive, n_off, flags;
  int s_off, s_cnt;   // session range [s_off, s_off + s_cnt) of a per-session launch
  int prefetch;       // the sets were built ahead of the gate (lfps_decode_prefetch, or
                      // beside it): the finish handles gated sessions and kappa = 0
                      // (every session; kappa = 0 is raised by the finish kernel)
  int epoch;          // call stamp in [1, 2^27): err[0] == epoch <=> this call failed
  const int* stamp;   // CUDA-graph steps: the stamp in device memory (set by the
                      // step's first kernel), used instead of epoch
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
  double* thr_next;   // [NS, 2, 4] thresholds of the upcoming select (stats -> select)
  int* counts;
  uint32_t* bits;
  int* probe_idx;
  float* probe_score;
  int* c2_idx;
  float* c2_score;
  double* uw;       // [NS, list_cap] scratch (exact top-k overflow)
  long long* trace; // [NS, 16] phase timestamps (LFPS_FLAG_TRACE)
  unsigned* done;     // [1] CTAs finished in the commit kernel (last one bumps n_ctx)
  int2* hot;          // [2 NS][16 nblk + 1] per-step C0 words (k_select.cu)
  double* scratch;
  BlockWs bw;
  // block-table KV (lfps_state.block_table): row r of unit (b, h) lives at
  // pool row (bt[b][r >> bs_shift] << bs_shift | r & bs_mask) * Hkv + h of a
  // [blocks, block_rows, Hkv, d] pool; bt == nullptr: contiguous [B, Hkv, n_max, d]
  const int* bt;
  int bs_shift, bs_mask, max_blocks;
};

// CNT_BLOCKS: table blocks the select kernel read (rebuilt + hot), a diagnostic
enum { CNT_C0 = 0, CNT_C1, CNT_PROBE, CNT_DROP, CNT_K, CNT_C2, CNT_CLAMP, CNT_BLOCKS, CNT_N };

// Row r of unit (b, h) -> its row number in the K / V buffers (row = d
// elements): the unit's contiguous span, or the block table's block.
// MODE 0: contiguous only; 1: block table only; 2: decided per call
// (c.bt), for the kernels off the hot path.
template <int MODE>
struct RowMapT {
  const int* bt;      // this request's block-table row (block table mode)
  int base;           // first row of the unit (contiguous), or h (block table)
  int shift, mask, hkv;
  __device__ __forceinline__ RowMapT(const Ctx& c, int b, int h) {
    shift = c.bs_shift; mask = c.bs_mask; hkv = c.Hkv;
    if (MODE == 1 || (MODE == 2 && c.bt)) {
      bt = c.bt + (size_t)b * c.max_blocks;
      base = h;
    } else {
      bt = nullptr;
      base = (b * c.Hkv + h) * c.n_max;
    }
  }
  __device__ __forceinline__ int operator()(int r) const {
    if (MODE == 0 || (MODE == 2 && !bt)) return base + r;
    return ((__ldg(bt + (r >> shift)) << shift) | (r & mask)) * hkv + base;
  }
};
using RowMap = RowMapT<2>;

__device__ __forceinline__ const __nv_bfloat16* krow(const Ctx& c, int b, int h, int i) {
  return c.K + (size_t)RowMap(c, b, h)(i) * c.d;
}
__device__ __forceinline__ const __nv_bfloat16* vrow(const Ctx& c, int b, int h, int i) {
  return c.V + (size_t)RowMap(c, b, h)(i) * c.d;
}

// err[1 + s] = (call stamp << 4) | code: a code counts only for the call whose
// stamp err[0] holds, so no kernel has to clear the codes before the gate and
// the stats kernel (which run concurrently) may raise them
__device__ __forceinline__ int call_stamp(const Ctx& c) {
  const int* p = c.stamp;
  const int e = c.epoch;
  return p ? __ldcg(p) : e;
}
__device__ __forceinline__ int err_code(const Ctx& c, int code) { return (call_stamp(c) << 4) | code; }
__device__ __forceinline__ void set_err(const Ctx& c, int s, int code) {
  const int ep = call_stamp(c);
  c.err[1 + s] = (ep << 4) | code;
  atomicExch(c.err, ep);
}

// phase timestamps (LFPS_FLAG_TRACE): slot k of session s = clock64() - t0;
// slot 15 / 14 hold the globaltimer at select entry / finish exit
__device__ __forceinline__ long long now_clk() { return clock64(); }
__device__ __forceinline__ long long now_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_at(const Ctx& c, int s, int slot, long long t0) {
  if ((c.flags & LFPS_FLAG_TRACE) && threadIdx.x == 0) c.trace[(size_t)s * 16 + slot] = now_clk() - t0;
}

__device__ __forceinline__ double* ver_row(const Ctx& c, int s) { return c.ver + (size_t)s * c.m_cap; }
__device__ __forceinline__ double* sla_row(const Ctx& c, int s) { return c.sla + (size_t)s * c.sla_cap; }

// LFPS_EARLY_TRIGGER: stats / select / finish let their dependents be
// scheduled from their start (the dependents still wait in pdl_wait for the
// whole grid), so the next kernel's CTAs fill the SMs during the last wave
#ifndef LFPS_EARLY_TRIGGER
#define LFPS_EARLY_TRIGGER 0
#endif

// ---- host-side launch wrappers (defined in the k_*.cu files) -------------
// Launch with programmatic stream serialization (PDL): the kernel may be
// scheduled while its predecessor in the stream drains; it calls pdl_wait()
// before reading anything the predecessor wrote.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// One-time setup of a launch site per device (cudaFuncSetAttribute is a
// per-device property): thread-safe, and redone on every device a launch
// site is first used on.  Racing first calls both run f (idempotent).
struct DeviceOnce {
  unsigned long long done[4] = {0ull, 0ull, 0ull, 0ull};   // 256 devices
  template <typename F>
  cudaError_t run(F f) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    unsigned long long* w = &done[(dev >> 6) & 3];
    const unsigned long long bit = 1ull << (dev & 63);
    if (__atomic_load_n(w, __ATOMIC_ACQUIRE) & bit) return cudaSuccess;
    e = f();
    if (e == cudaSuccess) __atomic_fetch_or(w, bit, __ATOMIC_RELEASE);
    return e;
  }
};

cudaError_t launch_gate(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st);
cudaError_t launch_stats(const Ctx& c, cudaStream_t st);
cudaError_t launch_select(const Ctx& c, int m_max, cudaStream_t st);
cudaError_t launch_topk(const Ctx& c, int implicit_base, cudaStream_t st);
cudaError_t launch_attend(const Ctx& c, const __nv_bfloat16* q, int exact_mode, cudaStream_t st);
cudaError_t launch_update(const Ctx& c, const __nv_bfloat16* k_new, const __nv_bfloat16* v_new,
                          cudaStream_t st);
cudaError_t launch_finish(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st);
cudaError_t launch_boot_tables(const Ctx& c, const float* w, int s_begin, int count, int m0,
                               cudaStream_t st);
cudaError_t launch_boot_stats(const Ctx& c, const __nv_bfloat16* q, int m_max, int b0, int nb,
                              cudaStream_t st);
cudaError_t launch_exact_score(const Ctx& c, const __nv_bfloat16* q, int m_max, cudaStream_t st);
cudaError_t launch_overlap(const Ctx& c, const int* sel, const int* sel_cnt, const int* ex,
                           const int* ex_cnt, int list_stride, int cnt_stride, double* eta,
                           cudaStream_t st);
cudaError_t launch_clear_err(const Ctx& c, cudaStream_t st);
cudaError_t launch_step_begin(const Ctx& c, cudaStream_t st);

// per-head stage API (k_stages.cu), fp64
cudaError_t stage_logits(const double* keys, int d, const int64_t* rows, int nrows, const double* q,
                         double* out, cudaStream_t st);
cudaError_t stage_thresholds(const double* ver, const double* sla, int m, double scale, double a,
                             int materialize, double* out, double* scratch, cudaStream_t st);
cudaError_t stage_candidates(int mode, const double* ver, const double* sla, int m, double scale,
                             const double* thr, const int64_t* in_idx, int n_in, const int* offsets,
                             int n_off, long long base_index, int n, int sink, int window,
                             int64_t* out_idx, int* out_count, cudaStream_t st);
cudaError_t stage_topk(const int64_t* idx, const double* scores, int p, int k, int64_t* out_idx,
                       int* out_count, cudaStream_t st);
cudaError_t stage_attend(const double* keys, const double* values, int d, const int64_t* idx,
                         int nidx, const double* q, double* out, double* weights, int* err,
                         cudaStream_t st);
cudaError_t stage_update(double* ver, double* sla, int base, int m, const int64_t* sel,
                         const double* w, int k, int renorm, double rf, double scale,
                         long long* clamps, double* tmp, cudaStream_t st);
cudaError_t stage_grow(double* ver, double* sla, int base, int m, int carry, cudaStream_t st);
cudaError_t stage_init_tables(const double* w, int s, int m, double r, double* ver, double* sla,
                              cudaStream_t st);
cudaError_t stage_head_stats(const double* keys, const double* values, int n, int d, int sink,
                             const double* q, double* mean_key, double* mean_value, double* sigma,
                             double* logit_tmp, int* err, cudaStream_t st);
cudaError_t stage_gate(const double* keys, const double* values, int n, int d, int sink, int window,
                       const double* q, const double* mean_key, const double* mean_value,
                       double sigma, int bypass_mode, double* out, int* err, cudaStream_t st);

}  // namespace lfps
