// k_finish.cu -- the per-session back half of a decode step in ONE kernel:
// candidate scoring (K3), Top-k (K4), sparse attention (K5) and the data
// checks feeding the tracker update (K6; the weights are computed and the
// update committed by k_update.cu once every session has passed).  One
// 256-thread CTA per (request, q-head) session.
//
//   rows     K / V rows stream through shared memory in tiles of 64 rows
//            (two per 8-lane group), 2 stages deep, gathered with cp.async
//            (16 B per thread, L2 only): no registers hold in-flight data;
//            64 KB per CTA -> 3 CTAs / SM.  (Per-row TMA bulk copies were
//            measured 2x slower: one 256-B request per row saturates the SM's
//            TMA unit; 3 stages at 2 CTAs / SM measured slower than 2 at 3.)
//   scores   z_j = (K[j] . q) / fp32(sqrt d) in the canonical order of
//            devmath.sdot32 (engine.py:168-170): 8 lanes per row, lane l
//            owns partials l and l + 8 (d/16 contiguous elements each, two
//            chains of fma.rn.f32.bf16 -- no bf16 widening), fold 8
//            (in-lane), 4, 2, 1 (shuffles; the group's two rows share them
//            in a reduce-scatter), IEEE division
//   top-k    k = max(1, round_half_even(frac * n)) (engine.py:167); if
//            k >= |probe| C2 = probe and scores + attention are ONE pass
//            over the rows; else all scores first, an MSB-first 4 x 8-bit
//            radix select of the k-th largest key with lowest-index ties
//            (topk_from_scores, attention.py:34-47), then the attention pass
//   attend   joint softmax over [sink logits, C2 logits] and sum w V
//            (engine.py:173-181): every 8-lane group keeps an online
//            (max, sum, acc) over its rows in the base-2 domain (MUFU.EX2,
//            packed fp32x2 FMAs), the 32 group states are merged at the end
//            (fp32)
//   checks   sinks and C2 scores finite (softmax_weights, numerics.py:61-62,
//            called at engine.py:177 and :184); the C2 max goes to wstat,
//            from which k_update.cu forms u = canonical fp64 softmax of the
//            C2 scores (devmath.softmax_update) and checks |sum u - 1| <=
//            1e-6 (tables.py:161-163)
#include "finish.cuh"

namespace lfps {

namespace {

using namespace fin;

// RM: the row mapping (RowMapT) -- 0 contiguous cache, 1 block table
template <int PQ, int RM>
__global__ void __launch_bounds__(kThreads, kRowCtas) lfps_finish_kernel(Ctx c, const __nv_bfloat16* q) {
  extern __shared__ __align__(128) uint8_t stages[];      // kStagesR x [K tile | V tile]
  __shared__ FinishShared sh;
  pdl_wait();                                             // the select kernel's lists
  if (LFPS_EARLY_TRIGGER) pdl_trigger();
  finish_session<PQ, RM>(c, q, c.s_off + blockIdx.x, stages, sh);
  if (!LFPS_EARLY_TRIGGER) pdl_trigger();
}

template <int PQ, int RM>
cudaError_t launch_finish_rm(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  const size_t smem = rows_smem(c.d);
  static DeviceOnce once;
  cudaError_t e = once.run([&] {
    cudaError_t r = cudaFuncSetAttribute(lfps_finish_kernel<PQ, RM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(lfps_finish_kernel<PQ, RM>,
                               cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    return r;
  });
  if (e != cudaSuccess) return e;
  return launch_pdl(lfps_finish_kernel<PQ, RM>, dim3(c.s_cnt), dim3(kThreads), smem, st, c, q);
}

template <int PQ>
cudaError_t launch_finish_d(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  return c.bt ? launch_finish_rm<PQ, 1>(c, q, st) : launch_finish_rm<PQ, 0>(c, q, st);
}

}  // namespace

cudaError_t launch_finish(const Ctx& c, const __nv_bfloat16* q, cudaStream_t st) {
  switch (c.d) {
    case 32: return launch_finish_d<2>(c, q, st);
    case 64: return launch_finish_d<4>(c, q, st);
    case 128: return launch_finish_d<8>(c, q, st);
    case 256: return launch_finish_d<16>(c, q, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace lfps
