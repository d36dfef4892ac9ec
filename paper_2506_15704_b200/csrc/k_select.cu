// k_select.cu -- thresholds and candidate construction (K1 + K2) from
// PERSISTENT block summaries, as two kernels:
//
//   lfps_stats_kernel   one 128-thread CTA per (session, table): A + B + C
//                       (tables.cuh maintain_table); runs beside the gate
//   lfps_select_kernel  one 256-thread CTA per session: C0 assembly + D
//                       (select.cuh select_session)
//
// Restates compute_thresholds (tables.py:295-317, _phys_moments :127-140),
// select_initial (candidates.py:45-58), expand (:61-82) and
// finalize_probe_set (:85-100).
//
// Each table is cut into 512-slot blocks of table slots (vertical: slot =
// logical index; slash: slot = sla_base + logical index, a window that only
// grows at its ends).  Every block carries a summary of its part of the
// window: the canonical segment moments (mean, M2, M3, M4) and the maximum
// phys value.  A decode step changes a table only at its C2 slots and at the
// one slot it grows by (k_update.cu marks those blocks dirty), and the lazy
// scale leaves phys values alone, so the summaries of all other blocks stay
// exact.  Per step
//
//   A  rebuilds the dirty blocks (every block when the session's summaries
//      are not valid: first step, after a renormalisation);
//   B  merges the window's segment moments in the canonical pairwise tree
//      (devmath.table_moments) -> tau, mean, degenerate, kappa in thr_next[];
//      exactly the same arithmetic as rebuilding every block;
//   C  the table's part of C0 = {slots with phys > tau / scale}: only "hot"
//      blocks (max above the threshold) can hold members, and only those are
//      read; their C0 words are listed in ws.hot, and the select kernel ORs
//      both tables' words into its bitmap;
//   D  C1 = F & dilate(C0, offsets), F read at dilated slots only;
//      probe = C1 | local tail, compacted into a sorted absolute index list.
//
// A, B and C are fp64 latency chains per table: running them per (session,
// table) in 128-thread CTAs (7 per SM) nearly doubles the sessions in flight over
// one 256-thread CTA per session doing both tables.
//
// All comparisons are exact fp64 (on bit patterns: phys values are +0 or
// positive).  Table bytes read per step: dirty + hot blocks, not 2 m.
#include "common.cuh"
#include "canon.cuh"
#include "ptx.cuh"
#include "tables.cuh"
#include "select.cuh"

namespace lfps {

namespace {

using namespace tbl;
using namespace sel;

#ifndef LFPS_STATS_CTAS
#define LFPS_STATS_CTAS 7
#endif
#ifndef LFPS_SELECT_CTAS
#define LFPS_SELECT_CTAS 5
#endif
constexpr int kStatsThreads = 128;

// A + B + C of one (session, table) by one 128-thread CTA (tables.cuh).
// valid[s]: 0 = rebuild every block, 1 = the summaries are current (rebuild
// the dirty blocks), 2 = thresholds and C0 words are current as well
// (nothing to do; reserved for an eager maintainer -- measured slower when
// fused into the update kernel).
__global__ void __launch_bounds__(kStatsThreads, LFPS_STATS_CTAS) lfps_stats_kernel(Ctx c) {
  __shared__ StatsShared sh;
  const int s = c.s_off + (blockIdx.x >> 1), t = blockIdx.x & 1;
  const int tid = threadIdx.x;
  if (LFPS_EARLY_TRIGGER) pdl_trigger();
  if (c.exhaustive) return;
  const int b = s / c.Hq;
  const int dw = c.bw.dwords;
  // independent prologue loads, issued together.  The stats kernel runs
  // concurrently with the gate, so it works for every session, gated or not.
  const int n = c.n_ctx[b];
  const int base = t ? c.sla_base[s] : 0;
  const int valid = c.bw.valid[s];
  const double sc = c.scale[s];
  uint32_t* dp = c.bw.dirty + (size_t)(2 * s + t) * dw + tid;
  const uint32_t dbits = tid < dw ? *dp : 0u;
  if (valid >= 2) return;                             // kept current by the update kernel
  if (tid < dw && dbits) *dp = 0u;
  const Window w = make_window(base, n - c.S);
  const long long tclk0 = now_clk();
  if ((c.flags & LFPS_FLAG_TRACE) && tid == 0 && t == 0) c.trace[(size_t)s * 16 + 15] = now_ns();
  maintain_table(c, s, t, w, sc, valid == 0, [&](int) { return dbits; }, sh, tid, 1, tclk0);
}

// C + D of one session (select.cuh).
__global__ void __launch_bounds__(kThreads, LFPS_SELECT_CTAS) lfps_select_kernel(Ctx c) {
  extern __shared__ __align__(16) uint32_t smem[];
  __shared__ SelectShared sh;
  pdl_wait();                                  // the stats kernel's thresholds and C0 words
  if (LFPS_EARLY_TRIGGER) pdl_trigger();
  select_session(c, c.s_off + blockIdx.x, smem, sh);
  if (!LFPS_EARLY_TRIGGER) pdl_trigger();
}

}  // namespace

cudaError_t launch_stats(const Ctx& c, cudaStream_t st) {
  lfps_stats_kernel<<<2 * c.s_cnt, kStatsThreads, 0, st>>>(c);
  return cudaGetLastError();
}

cudaError_t launch_select(const Ctx& c, int m_max, cudaStream_t st) {
  const size_t smem = select_smem(m_max);
  static DeviceOnce once;
  cudaError_t e = once.run([] {
    cudaError_t r = cudaFuncSetAttribute(lfps_select_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (r == cudaSuccess)
      r = cudaFuncSetAttribute(lfps_select_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    return r;
  });
  if (e != cudaSuccess) return e;
  return launch_pdl(lfps_select_kernel, dim3(c.s_cnt), dim3(kThreads), smem, st, c);
}

}  // namespace lfps
