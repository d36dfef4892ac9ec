// finish.cuh -- the per-session back half of a decode step (see k_finish.cu),
// as a device function shared by the per-session and per-unit kernels.
#pragma once

#include "rows.cuh"

namespace lfps {
namespace fin {

using namespace rows;

struct FinishShared {
  float sink_z[32];
  float part_m[kGroups8];
  float part_s[kGroups8];
  float gmax[kWarps];
  double red[16];
  int warp_sums[kWarps];
  unsigned hist[256];
  unsigned sel_digit;
  int sel_want;
};

// Merge the 32 group states of `at` into out[s], then the data checks (chk:
// NaN once a score was not finite) and the C2 max for the update weights.
// stages: scratch (>= 2 * 32 * d floats).
template <int PQ>
__device__ __forceinline__ void finish_tail(const Ctx& c, int s, uint8_t* stages, FinishShared& sh,
                                            const Attn<PQ>& at, float chk, float mxc, long long t0) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5, l8 = tid & 7, grp = tid >> 3;
  trace_at(c, s, 8, t0);
  // ---- merge the 32 group states into the output (stages reused as scratch) ----------
  {
    constexpr int D = PQ * 16;
    constexpr int kG = kThreads / D;                    // threads per output element
    constexpr int kPer = kGroups8 / kG;                 // groups each of them merges
    float* part = reinterpret_cast<float*>(stages);     // [kGroups8][D]
#pragma unroll
    for (int e = 0; e < PQ; ++e) {
      part[grp * D + l8 * PQ + e] = at.acc[e].x;
      part[grp * D + (l8 + 8) * PQ + e] = at.acc[e].y;
    }
    if (l8 == 0) { sh.part_m[grp] = at.m; sh.part_s[grp] = at.s; }
    __syncthreads();
    float M = -INFINITY;
#pragma unroll 8
    for (int x = 0; x < kGroups8; ++x) M = fmaxf(M, sh.part_m[x]);
    const int t = tid % D, g = tid / D;
    float num = 0.0f, den = 0.0f;
#pragma unroll
    for (int xi = 0; xi < kPer; ++xi) {
      const int x = g * kPer + xi;
      if (sh.part_m[x] == -INFINITY) continue;
      const float f = ex2(sh.part_m[x] - M);
      num = fmaf(f, part[x * D + t], num);
      den = fmaf(f, sh.part_s[x], den);
    }
    __syncthreads();                                     // part is reused below
    part[g * D + t] = num;
    part[kG * D + g * D + t] = den;
    __syncthreads();
    if (tid < D) {
      float nsum = 0.0f, dsum = 0.0f;
#pragma unroll
      for (int x = 0; x < kG; ++x) {
        nsum += part[x * D + tid];
        dsum += part[kG * D + x * D + tid];
      }
      c.out[(size_t)s * c.d + tid] = nsum / dsum;
    }
  }

  trace_at(c, s, 9, t0);
  // ---- data checks; the C2 max for the update weights (k_update.cu) ----------------
  if (__syncthreads_or(!(chk == 0.0f))) {
    if (tid == 0) set_err(c, s, LFPS_ERR_NONFINITE_SCORES);
    return;
  }
  for (int o = 16; o >= 1; o >>= 1) mxc = fmaxf(mxc, __shfl_xor_sync(LFPS_FULL, mxc, o));
  if (lane == 0) sh.gmax[warp] = mxc;
  __syncthreads();
  if (tid == 0) {
    float mf = sh.gmax[0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) mf = fmaxf(mf, sh.gmax[w]);
    c.bw.wstat[2 * (size_t)s] = (double)mf;
    if (c.flags & LFPS_FLAG_TRACE) {
      c.trace[(size_t)s * 16 + 10] = now_clk() - t0;
      c.trace[(size_t)s * 16 + 14] = now_ns();
    }
  }
}

// The whole back half of one session's step, run by a 256-thread CTA.
// `stages` is kStagesR x [K tile | V tile] of dynamic shared memory.
template <int PQ, int RM>
__device__ __forceinline__ void finish_session(const Ctx& c, const __nv_bfloat16* q, int s,
                                               uint8_t* stages, FinishShared& sh) {
  const int tid = threadIdx.x;
  const int l8 = tid & 7;
  const int b = s / c.Hq, h = (s % c.Hq) / c.G;
  const int n = c.n_ctx[b];
  const int S = c.S;
  int* cnt = c.counts + (size_t)s * CNT_N;

  if (c.bypass[s]) {
    if (tid == 0) {
      cnt[CNT_K] = 0; cnt[CNT_C2] = 0; cnt[CNT_CLAMP] = 0;
      // a prefetched select built this session's sets before the gate ran
      if (c.prefetch) { cnt[CNT_C0] = 0; cnt[CNT_C1] = 0; cnt[CNT_PROBE] = 0; cnt[CNT_DROP] = 0; }
    }
    return;
  }
  if (c.prefetch && tid < 2 && !c.exhaustive) {
    // kappa = 0 (tables.py:314-315) fails a non-bypassed step only; the
    // prefetched select exported the thresholds instead of raising it
    const double* th = c.thr + (size_t)(2 * s + tid) * 4;
    if (th[2] == 0.0 && th[3] == 0.0) set_err(c, s, LFPS_ERR_KAPPA_ZERO);
  }
  const int p = cnt[CNT_PROBE];
  const long long t0 = now_clk();
  if ((c.flags & LFPS_FLAG_TRACE) && tid == 0) c.trace[(size_t)s * 16 + 13] = now_ns();
  const int* pidx = c.probe_idx + (size_t)s * c.list_cap;
  float* pz = c.probe_score + (size_t)s * c.list_cap;
  // contiguous cache: the unit's base in registers and unit-local rows
  // (parameter-bank bases get rematerialised inside the row loop);
  // block table: the pool base and pool rows
  const __nv_bfloat16* kb = RM == 0 ? krow(c, b, h, 0) : c.K;
  const __nv_bfloat16* vb = RM == 0 ? vrow(c, b, h, 0) : c.V;
  const RowMapT<RM> rmap(c, b, h);
  auto rm = [&](int r) { return RM == 0 ? r : rmap(r); };
  const Part<PQ> qp = ld_part<PQ>(q + (size_t)s * c.d, l8);   // packed bf16 partials of q
  int k = (int)rint(c.frac * (double)n);
  if (k < 1) k = 1;
  int* c2i = c.c2_idx + (size_t)s * c.list_cap;
  float* c2z = c.c2_score + (size_t)s * c.list_cap;
  const int k2 = k >= p ? p : k;
  if (tid == 0) { cnt[CNT_K] = k; cnt[CNT_C2] = k2; }

  Attn<PQ> at;
  at.init();
  float chk = 0.0f;                                     // NaN once any score is not finite
  float mxc = -INFINITY;                                // max C2 score of this group
  float* c2zS = c2z - S;                                // indexed by list entry rid >= S
  float* pzS = pz - S;
  const int* pidxS = pidx - S;

  if (k >= p) {
    // ---- C2 = probe (the common case): score and attend in ONE pass ---------------------
    // a C2 / sink score: each lane keeps the row it folded in the
    // reduce-scatter (lanes 0-3 row a, 4-7 row b), lanes 0 and 4 store it
    auto keep = [&](int rid, float z) {
      chk = __fmaf_rn(z, 0.0f, chk);
      if (rid >= S) {
        mxc = fmaxf(mxc, z);
        if ((l8 & 3) == 0) c2zS[rid] = z;
      } else if ((l8 & 3) == 0) {
        sh.sink_z[rid] = z;
      }
    };
    stream_rows<kFused, PQ>(
        stages, kb, vb, S + p, [&](int rid) { return rm(rid < S ? rid : __ldg(pidxS + rid)); },
        [&](const Rows2& r) {
          const float2 z = score_rows<PQ>(r, qp, c.sqrt_d_f32);
          {
            const bool b4 = (l8 & 4) != 0;
            if (b4 ? r.ok[1] : r.ok[0]) keep(b4 ? r.rid[1] : r.rid[0], b4 ? z.y : z.x);
          }
          if (r.ok[1]) {
            at.absorb2(z.x * kLog2e, ld_part_s<PQ>(r.v[0], l8), z.y * kLog2e, ld_part_s<PQ>(r.v[1], l8));
          } else if (r.ok[0]) {
            at.absorb(z.x * kLog2e, ld_part_s<PQ>(r.v[0], l8));
          }
        });
    for (int j = tid; j < p; j += kThreads) c2i[j] = __ldg(pidx + j);
  } else {
    // ---- scores of the sinks and the probe rows -------------------------------------------
    stream_rows<kScore, PQ>(
        stages, kb, vb, S + p, [&](int rid) { return rm(rid < S ? rid : __ldg(pidxS + rid)); },
        [&](const Rows2& r) {
          const float2 z = score_rows<PQ>(r, qp, c.sqrt_d_f32);
          if (l8 == 0) {
#pragma unroll
            for (int i = 0; i < kR; ++i) {
              if (!r.ok[i]) continue;
              const float zi = i ? z.y : z.x;
              if (r.rid[i] < S) sh.sink_z[r.rid[i]] = zi;
              else pzS[r.rid[i]] = zi;
            }
          }
        });
    // ---- Top-k: MSB-first radix select of the k-th largest key ---------------------------
    uint32_t prefix = 0, mask = 0;
    int want = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
      sh.hist[tid] = 0;
      __syncthreads();
      for (int j = tid; j < p; j += kThreads) {
        const uint32_t key = score_key(pz[j]);
        if ((key & mask) == prefix) atomicAdd(&sh.hist[(key >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (tid < 32) {
        unsigned loc = 0;
#pragma unroll
        for (int t = 0; t < 8; ++t) loc += sh.hist[255 - 8 * tid - t];
        unsigned incl = loc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const unsigned y = __shfl_up_sync(LFPS_FULL, incl, o);
          if (tid >= o) incl += y;
        }
        const unsigned excl = incl - loc;
        if (excl < (unsigned)want && incl >= (unsigned)want) {
          unsigned cum = excl;
          for (int t = 0; t < 8; ++t) {
            const unsigned dgt = 255 - 8 * tid - t;
            const unsigned hc = sh.hist[dgt];
            if (cum + hc >= (unsigned)want) {
              sh.sel_digit = dgt;
              sh.sel_want = want - (int)cum;
              break;
            }
            cum += hc;
          }
        }
      }
      __syncthreads();
      prefix |= sh.sel_digit << shift;
      mask |= 255u << shift;
      want = sh.sel_want;
      __syncthreads();
    }
    const uint32_t kth = prefix;
    const int need_eq = want;
    int out_n = 0, eq_seen = 0;
    for (int t0 = 0; t0 < p; t0 += kThreads) {
      const int j = t0 + tid;
      const uint32_t key = j < p ? score_key(pz[j]) : 0u;
      const int gt = (j < p) && key > kth;
      const int eq = (j < p) && key == kth;
      int eq_tot, take_tot;
      const int eq_before = scan256(eq, sh.warp_sums, &eq_tot);
      const int take = gt || (eq && eq_seen + eq_before < need_eq);
      const int pos = scan256(take, sh.warp_sums, &take_tot);
      if (take) {
        c2i[out_n + pos] = pidx[j];
        c2z[out_n + pos] = pz[j];
      }
      out_n += take_tot;
      eq_seen += eq_tot;
    }
    __syncthreads();
    // ---- attention over sinks u C2 ------------------------------------------------------
    auto zof = [&](int rid) {
      const float z = rid < S ? sh.sink_z[rid] : c2zS[rid];
      chk = __fmaf_rn(z, 0.0f, chk);
      if (rid >= S) mxc = fmaxf(mxc, z);
      return z * kLog2e;
    };
    stream_rows<kAttend, PQ>(
        stages, kb, vb, S + k2, [&](int rid) { return rm(rid < S ? rid : c2i[rid - S]); },
        [&](const Rows2& r) {
          if (r.ok[1]) {
            const float za = zof(r.rid[0]), zb = zof(r.rid[1]);
            at.absorb2(za, ld_part_s<PQ>(r.v[0], l8), zb, ld_part_s<PQ>(r.v[1], l8));
          } else if (r.ok[0]) {
            at.absorb(zof(r.rid[0]), ld_part_s<PQ>(r.v[0], l8));
          }
        });
  }

  finish_tail<PQ>(c, s, stages, sh, at, chk, mxc, t0);
}

}  // namespace fin
}  // namespace lfps
