/*
 * lfps_b200.h -- C-ABI of the B200-native LFPS decode-step library
 * (liblfps_b200.so, sm_100a).
 *
 * The reference (arXiv 2506.15704, pkg/src/lfps) is a pure Python/numpy
 * package with no FFI: its drop-in surface is the Python functions
 *   prefill_bootstrap  engine.py:67-94
 *   decode_step        engine.py:97-201   (Algorithm 1, one head, one step)
 *   run_session        engine.py:204-219
 *   exact_topk_step    bench.py:73-80     (the exact comparison path)
 * re-exported by __init__.py:13-58.  These entry points are what those
 * functions become for a batch of (request, q-head) sessions on one GPU; the
 * Python package paper_2506_15704_b200 binds them with ctypes
 * (paper_2506_15704_b200/_lib.py) and mirrors the reference names on top.
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every pointer in lfps_state /
 *    lfps_workspace is a DEVICE pointer owned by the caller; the library
 *    never allocates, except the optional paged KV store (lfps_kv_pool_*),
 *    which owns its pages.  `stream` is a cudaStream_t passed as void*.
 *  - Return 0 on success or a negative LFPS_E_* code; lfps_last_error()
 *    returns a thread-local message for the last failure.  All argument
 *    validation happens on the host before any launch, so a rejected call
 *    leaves the state untouched (engine.py:111-120 "all computation before
 *    mutation").
 *  - Data-dependent failures the reference raises on (non-finite logits,
 *    gate.py:104-113; weights not summing to 1, tables.py:161-163; kappa == 0,
 *    the ZeroDivisionError of tables.py:315) are detected on the device: the
 *    step then commits NO state for any session (tables, KV rows and n_ctx
 *    unchanged) and err[0] holds the call's nonzero stamp (0 after a
 *    committed step); err[1 + s] = (stamp << 4) | code for the sessions that
 *    raised in that call (codes with another stamp are stale).  A negative
 *    err[0] marks the one failure detected only inside the commit (the
 *    weight-sum check, unreachable for finite scores): the other sessions
 *    commit, the KV rows and n_ctx advance, and the failed sessions' tables
 *    only grow (as on a gated step), so every table stays in step with its
 *    KV store.
 *  - Threading: calls on distinct workspaces (sessions) are reentrant; each
 *    workspace gets its own internal streams and events on its first decode
 *    step (lfps_workspace_release frees them).  One workspace is driven by
 *    one host thread at a time (the reference's single writer per session,
 *    engine.py:38-47).
 *  - Session index s = b * Hq + qh, q-head qh reads KV head qh / G (GQA).
 */
#ifndef LFPS_B200_H
#define LFPS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define LFPS_API __attribute__((visibility("default")))
#else
#define LFPS_API
#endif

#define LFPS_ABI_VERSION 9

#define LFPS_OK 0
#define LFPS_E_INVALID -1   /* bad argument (shape, range, capacity) */
#define LFPS_E_CUDA -2      /* CUDA runtime error */
#define LFPS_E_UNSUPPORTED -3

/* per-session device error codes (err[1 + s]) */
#define LFPS_ERR_NONFINITE_LOGITS 1   /* gate.py:104-106 */
#define LFPS_ERR_NONFINITE_RHO 2      /* gate.py:112-113 */
#define LFPS_ERR_KAPPA_ZERO 3         /* tables.py:314-315 ZeroDivisionError */
#define LFPS_ERR_WEIGHT_SUM 4         /* tables.py:161-163 */
#define LFPS_ERR_PREFILL_SUM 5        /* engine.py:84-86 */
#define LFPS_ERR_ZERO_QUERY 6         /* gate.py:61-63 zero-norm prefill query */
#define LFPS_ERR_NONFINITE_SCORES 7   /* numerics.py:61-62 via engine.py:177,184 */

/* Problem dimensions of one layer. */
typedef struct lfps_dims {
  int32_t batch;     /* B requests */
  int32_t kv_heads;  /* Hkv */
  int32_t group;     /* G query heads per KV head (Hq = Hkv * G) */
  int32_t d;         /* head dimension, multiple of 16, <= 256 */
  int32_t n_max;     /* KV rows allocated per (request, KV head) */
  int32_t m_cap;     /* vertical-table slots per session (even); the slash
                        table holds lfps_slash_capacity(dims) slots */
} lfps_dims;

/* LfpsConfig (config.py:11-42) plus the per-call budget. */
typedef struct lfps_params {
  double r;            /* decay */
  double epsilon;      /* gate threshold */
  double a;            /* threshold scale */
  double k_fraction;   /* Top-k budget fraction, (0, 1] */
  double sqrt_d;       /* math.sqrt(d) */
  float sqrt_d_f32;    /* fp32(sqrt(d)) used by the fp32 score dot */
  int32_t s;           /* prefill steps seeding the tables */
  int32_t sink_count;  /* S, <= 31 */
  int32_t local_window;/* L, <= 64 */
  int32_t bypass_mode; /* 0 = sink_average, 1 = mean_only */
  int32_t exhaustive;  /* exhaustive_fallback */
  int32_t n_offsets;   /* distinct expansion offsets, <= 16 */
  int32_t offsets[16]; /* each in [-31, 31] */
  int32_t flags;       /* LFPS_FLAG_* */
} lfps_params;

/* lfps_params.flags */
#define LFPS_FLAG_PREFETCHED 64  /* the step's candidate construction (thresholds,
                                    C0, C1, probe sets: stats + select) was run
                                    ahead by lfps_decode_prefetch on this
                                    workspace; the step runs the gate, the
                                    finish and the commit only */
#define LFPS_FLAG_GRAPH 16       /* enqueue a decode step as one CUDA-graph launch: the
                                    step is captured once per (shapes, params,
                                    state, workspace, device buffers, context
                                    bucket) and replayed; the call stamp is then
                                    drawn on the device (ws.done[1]) */
#define LFPS_FLAG_SPLIT 8        /* run two session halves' gate/select/finish on two
                                    internal streams (fork/join on the caller's) */
#define LFPS_FLAG_TRACE 2        /* per-session phase timestamps (clock64 deltas and
                                    globaltimer) of the select and finish kernels
                                    to ws.trace ([NS][16] int64) */
#define LFPS_FLAG_EXPORT_SETS 1  /* write the C0 / C1 bitmaps of every session to
                                    ws.bits ([NS][2][words]: C0 then C1) */

/* Persistent per-layer state (caller-owned device buffers). */
typedef struct lfps_state {
  void* k_cache;          /* bf16 [B, Hkv, n_max, d] */
  void* v_cache;          /* bf16 [B, Hkv, n_max, d] */
  int32_t* n_ctx;         /* [B] rows currently in the cache (incl. sinks) */
  double* ver;            /* [NS, m_cap] vertical phys table */
  double* sla;            /* [NS, slash_cap] slash phys table: logical index i
                             lives at slot sla_base + i.  The window only grows
                             (down by one per slash shift, up by one per gated
                             step), so it never wraps; slash_cap =
                             lfps_slash_capacity(dims) =
                             2 * (roundup(m_cap, 512) + 512) */
  double* scale;          /* [NS] lazy decay scale */
  int32_t* sla_base;      /* [NS] slot of slash logical index 0 */
  int64_t* clamp_count;   /* [NS] cumulative clamp counter */
  double* mean_key;       /* [B * Hkv, d] prior K-bar (gate.py:71) */
  double* mean_value;     /* [B * Hkv, d] prior V-bar (gate.py:72) */
  double* sigma_hat_sq;   /* [NS] prior sigma^2 / |q|^2 (gate.py:67-73) */
  /* Block-table KV (a serving caller's paged cache, vLLM-style): when
     block_table is not NULL, k_cache / v_cache are pools [blocks,
     block_rows, Hkv, d] and row r of (request b, KV head h) is pool row
     (block_table[b * max_blocks + r / block_rows] * block_rows +
     r % block_rows) * Hkv + h; block_rows is a power of two and n_max ==
     max_blocks * block_rows.  The caller owns the table: the blocks of rows
     [0, n_ctx[b] + 1) must be mapped before a decode step (the step appends
     row n_ctx[b]).  NULL: the contiguous [B, Hkv, n_max, d] layout. */
  const int32_t* block_table;
  int32_t block_rows;
  int32_t max_blocks;
} lfps_state;

/* Offsets (bytes) of every region inside one workspace buffer. */
typedef struct lfps_ws_layout {
  size_t total_bytes;
  size_t rho;         /* f64 [NS] sink share */
  size_t bypass;      /* i32 [NS] 1 if gated */
  size_t err;         /* i32 [1 + NS] err[0] = failed call's stamp, err[1+s]
                         = stamp << 4 | code per session */
  size_t out;         /* f32 [NS, d] attention output */
  size_t thr;         /* f64 [NS, 2, 4] tau, mean, degenerate, kappa per table */
  size_t counts;      /* i32 [NS, 8] |c0| |c1| |probe| c0_dropped k |c2| clamps
                         table-blocks-read */
  size_t bits;        /* u32 [NS, 2 tables, words] C0 bitmaps of fallback items */
  size_t probe_idx;   /* i32 [NS, list_cap] absolute indices, ascending */
  size_t probe_score; /* f32 [NS, list_cap] */
  size_t c2_idx;      /* i32 [NS, list_cap] */
  size_t c2_score;    /* f32 [NS, list_cap] */
  size_t uw;          /* f64 [NS, list_cap] scratch: exact-path top-k overflow */
  size_t scratch;     /* f64 [NS, list_cap] bootstrap scratch */
  /* Block summaries of the tracker tables.  These PERSIST across steps (a
     cache of the state, kept in the workspace): item = 2 s + table (0 =
     vertical, 1 = slash); block b covers table slots [512 b, 512 b + 512)
     intersected with the item's window.  A zero-filled workspace is valid:
     valid[s] == 0 makes the next step rebuild every block of session s. */
  size_t bsum;        /* f64 [2 NS, nblk, 4] segment mean, M2, M3, M4 */
  size_t bmax;        /* f64 [2 NS, nblk] segment max phys value */
  size_t dirty;       /* u32 [2 NS, dirty_words] blocks to rebuild */
  size_t valid;       /* i32 [NS] summaries of session s are current */
  size_t wstat;       /* f64 [NS, 2] max and normaliser of the update softmax */
  size_t trace;       /* i64 [NS, 16] phase timestamps (LFPS_FLAG_TRACE) */
  size_t done;        /* u32 [16]: [0] commit-kernel completion counter (kept at
                         0), [1] the call stamp of a CUDA-graph step */
  size_t hot;         /* i32x2 [2 NS, 16 nblk + 1] per-step C0 words of each
                         table: (count, table blocks read), then (logical
                         index of the word's first slot, slot bits) */
  size_t thr_next;    /* f64 [NS, 2, 4] thresholds computed for the select
                         kernel (copied to thr for the non-gated sessions) */
  int32_t nblk;       /* blocks per item (slash_cap / 512) */
  int32_t dirty_words;
  int32_t words;      /* bitmap words per (session, table, kind) */
  int32_t list_cap;   /* capacity of each per-session list (m_cap rounded up to 32) */
} lfps_ws_layout;

typedef struct lfps_workspace {
  void* base;         /* device buffer of layout.total_bytes */
  size_t bytes;
} lfps_workspace;

LFPS_API int lfps_abi_version(void);
LFPS_API const char* lfps_last_error(void);

/* Workspace layout for these dimensions. */
LFPS_API int lfps_workspace_layout(const lfps_dims* dims, lfps_ws_layout* out);

/* Slots of one session's slash table (>= 0; negative LFPS_E_* on bad dims). */
LFPS_API int lfps_slash_capacity(const lfps_dims* dims);

/* Release the internal streams and events the library keeps for a workspace
 * (created by its first decode step; each workspace has its own, so host
 * threads may step distinct sessions concurrently).  Waits for that
 * workspace's internal work; call before freeing the workspace buffer.
 * (No reference counterpart: HeadSession is garbage-collected state,
 * engine.py:38-47.) */
LFPS_API int lfps_workspace_release(const lfps_workspace* ws);

/* Seed the tracker tables of sessions [s_begin, s_begin + count) from their
 * trailing prefill weights (Eq. 4; init_tables, tables.py:247-281).
 * weights: f32 device [count, p.s, m0] with m0 = n_ctx[b] - S of each
 * session's request; rows must sum to 1 within 1e-4 (engine.py:84-86). */
LFPS_API int lfps_bootstrap_tables(const lfps_dims* dims, const lfps_params* p,
                          const lfps_state* st, const lfps_workspace* ws,
                          const float* weights, int32_t s_begin, int32_t count,
                          int32_t m0, void* stream);

/* Freeze the gate priors of every session from the prefill rows
 * (compute_head_stats, gate.py:51-74).  last_query: bf16 device [NS, d]. */
LFPS_API int lfps_bootstrap_stats(const lfps_dims* dims, const lfps_params* p,
                         const lfps_state* st, const lfps_workspace* ws,
                         const void* last_query, void* stream);
/* The same for requests [b_begin, b_begin + b_count) only (a request
 * (re)loaded into a running batch); the other requests' priors stay. */
LFPS_API int lfps_bootstrap_stats_requests(const lfps_dims* dims, const lfps_params* p,
                                           const lfps_state* st, const lfps_workspace* ws,
                                           const void* last_query, int32_t b_begin,
                                           int32_t b_count, void* stream);

/* One LFPS decode step for all B * Hq sessions (decode_step,
 * engine.py:97-201): gate, thresholds, candidates, fp32 probe scoring,
 * Top-k, joint sink+selection attention, table update, then KV append of
 * k_new / v_new and n_ctx += 1.  Table updates, the append and n_ctx are
 * committed by the last kernels of the step, after every data check of
 * every session has passed (err[0] != this call's stamp), so a failed step
 * changes nothing
 * but the block-summary cache (which stays consistent with the tables).
 * q: bf16 [B, Hq, d]; k_new, v_new: bf16 [B, Hkv, d]; all device.
 * n_host: the caller's host copy of n_ctx [B] (used for validation and
 * launch sizing; must match the device copy).  Results land in the
 * workspace (out, counts, c2 lists, rho, bypass, err). */
LFPS_API int lfps_decode_step(const lfps_dims* dims, const lfps_params* p,
                     const lfps_state* st, const lfps_workspace* ws,
                     const void* q, const void* k_new, const void* v_new,
                     const int32_t* n_host, void* stream);

/* lfps_decode_step plus the step's attention output copied to out_host
 * (f32 [B, Hq, d], host memory; pinned for an asynchronous copy) as soon as
 * the output is final: the copy runs on an internal stream alongside the
 * commit kernel, and the caller's stream waits for it, so out_host is
 * filled when the caller's stream reaches the end of the call.  A step that
 * fails a data check still copies its (partial) output. */
LFPS_API int lfps_decode_step_host_out(const lfps_dims* dims, const lfps_params* p,
                     const lfps_state* st, const lfps_workspace* ws,
                     const void* q, const void* k_new, const void* v_new,
                     const int32_t* n_host, void* out_host, void* stream);

/* The step with host inputs AND host output: in_host (host memory, pinned
 * for an asynchronous copy) holds the step's inputs packed as bf16
 * [q (B*Hq*d) | k_new (B*Hkv*d) | v_new (B*Hkv*d)]; they are copied to
 * in_dev (a device buffer of lfps_step_input_bytes(dims)) on an internal
 * stream that starts with the call, so the copy overlaps the step's table
 * statistics (which do not read the inputs) and only the gate waits for it.
 * in_dev must not be touched by other work until the caller's stream
 * reaches the end of the call.  out_host as lfps_decode_step_host_out, or
 * NULL for no output copy. */
LFPS_API int lfps_decode_step_host_io(const lfps_dims* dims, const lfps_params* p,
                     const lfps_state* st, const lfps_workspace* ws,
                     const void* in_host, void* in_dev, const int32_t* n_host,
                     void* out_host, void* stream);

/* The q-independent half of the next decode step, run ahead: the tracker
 * thresholds, C0, C1 and the probe sets of every session depend on the
 * tables and the context only (engine.py:146-160: compute_thresholds,
 * select_initial, expand, finalize_probe_set do not read q), so they can be
 * built while the caller still computes the step's queries (e.g. during the
 * previous layers of the model).  The next lfps_decode_step* call on this
 * workspace with LFPS_FLAG_PREFETCHED in its params then runs the gate, the
 * finish and the commit only; it must follow on the same stream (or after
 * an event) with the same dims, params (except k_fraction) and state, and
 * no other decode step may run on the workspace in between.  A session the
 * gate bypasses reports no candidates, as in the normal step; a kappa = 0
 * threshold (tables.py:314-315) fails the step only for a non-bypassed
 * session, as in the normal step.  Not captured as a CUDA graph. */
LFPS_API int lfps_decode_prefetch(const lfps_dims* dims, const lfps_params* p,
                                  const lfps_state* st, const lfps_workspace* ws,
                                  const int32_t* n_host, void* stream);

/* Block the calling host thread until the output of the last decode step
 * with a host output (lfps_decode_step_host_out / _host_io) on this workspace
 * is in host memory.  The step's commit (tracker update, KV append) may
 * still be running: an autoregressive loop needs only the output to build
 * the next step's queries, and the next step is ordered after the commit on
 * the stream anyway. */
LFPS_API int lfps_wait_output(const lfps_workspace* ws);

/* Bytes of the packed step input of lfps_decode_step_host_io (< 0: invalid
 * dims). */
LFPS_API int64_t lfps_step_input_bytes(const lfps_dims* dims);

/* Exact full-scan Top-k comparison path (exact_topk_step, bench.py:73-80)
 * over the pre-append rows of every session: fp32 scores of all non-sink
 * rows, Top-k with lower-index ties, joint sink+selection output.  Read-only
 * on the state; results in ws (c2 lists = the exact set, out). */
LFPS_API int lfps_exact_topk_step(const lfps_dims* dims, const lfps_params* p,
                         const lfps_state* st, const lfps_workspace* ws,
                         const void* q, const int32_t* n_host, void* stream);

/* Overlap ratio eta per session (overlap_ratio, attention.py:116-124):
 * |sel ∩ exact| / |exact| for two ascending index lists per session.
 * List s starts at sel + s * list_stride; its length is
 * sel_cnt[s * cnt_stride] (same for exact).  eta: f64 [NS]. */
LFPS_API int lfps_overlap(const lfps_dims* dims, const int32_t* sel, const int32_t* sel_cnt,
                 const int32_t* exact, const int32_t* exact_cnt, int32_t list_stride,
                 int32_t cnt_stride, double* eta, void* stream);

/* Per-kernel CUDA-event timing.  While enabled, every kernel the entry
 * points launch is bracketed by events on its stream (do not enable during
 * CUDA-graph capture).  lfps_profile_collect waits for the events, sums the
 * durations per kernel name into out[0, *n_out) and clears the record. */
typedef struct lfps_kernel_time {
  char name[32];
  int32_t launches;
  double total_ms;
} lfps_kernel_time;
LFPS_API int lfps_profile_enable(int on);
LFPS_API int lfps_profile_collect(lfps_kernel_time* out, int32_t cap, int32_t* n_out);

/* Number of kernels lfps_decode_step launches for these dims and params
 * flags (dims may be NULL: the serial sequence), and lfps_exact_topk_step. */
LFPS_API int lfps_decode_launches(const lfps_dims* dims, int32_t flags);
LFPS_API int lfps_exact_launches(void);

/* Paged KV store (a paged-KV caller).  The kernels address
 * K/V as lfps_state.k_cache / v_cache [B, Hkv, n_max, d]; the pool reserves
 * that range as VIRTUAL address space on the current device and backs it
 * with physical pages (the device's allocation granularity, 2 MiB) only
 * where a (request, KV head) has rows, so the decode kernels see the
 * contiguous layout with no page table while memory follows the live
 * contexts.  Every (request, KV head) span n_max * d * 2 bytes must be a
 * multiple of the page size: lfps_kv_pool_page_bytes() gives it.
 * lfps_kv_pool_reserve backs rows [0, rows + 64) of one (request, KV head)
 * (the 64-row slack covers the last row tile of any kernel), mapping pages
 * as the context grows; lfps_kv_pool_release unmaps all of request b's
 * pages (a finished request).  The reference keeps one KvStore per head
 * that doubles and copies when full (store.py:8-90, _grow at :79-90); here
 * growth maps one more page, without a copy. */
typedef struct lfps_kv_pool lfps_kv_pool;
LFPS_API int64_t lfps_kv_pool_page_bytes(void);
LFPS_API int lfps_kv_pool_create(const lfps_dims* dims, lfps_kv_pool** pool,
                                 void** k_cache, void** v_cache);
LFPS_API int lfps_kv_pool_reserve(lfps_kv_pool* pool, int32_t b, int32_t h, int64_t rows);
LFPS_API int lfps_kv_pool_release(lfps_kv_pool* pool, int32_t b);
LFPS_API int64_t lfps_kv_pool_mapped_bytes(const lfps_kv_pool* pool);
LFPS_API int lfps_kv_pool_destroy(lfps_kv_pool* pool);

/* ---- Per-head stage API (k_stages.cu) ---------------------------------
 * The reference also exposes each stage of the decode step on its own, on
 * one head's float64 state (pkg/src/lfps/__init__.py:13-58).  These entry
 * points are those stages on the device at the reference's precision: fp64
 * K/V rows [n, d] (any d >= 1), fp64 tables, fp64 logits and softmax.  All
 * arrays are device pointers; indices are int64 absolute positions unless
 * stated; sets are sorted and unique.  One kernel launch each, on `stream`;
 * argument checks on the host before the launch.  Data errors the reference
 * raises are returned in a device int (*err) with the per-session codes
 * above (LFPS_ERR_*). */

/* row_logits (numerics.py:33-49): out[i] = keys[rows[i]] . q / sqrt(d);
 * rows NULL = rows 0 .. nrows-1. */
LFPS_API int lfps_stage_logits(const double* keys, int32_t d, const int64_t* rows, int32_t nrows,
                               const double* q, double* out, void* stream);
/* compute_thresholds (tables.py:295-317), or thresholds_oracle (:320-331)
 * with materialize = 1, of ver[0, m) and sla[0, m) (phys values; sla points
 * at logical slot 0) at lazy scale `scale`: out[7] = tau_v, mean_v, deg_v,
 * tau_s, mean_s, deg_s, then 3 if kappa == 0 (ZeroDivisionError) else
 * untouched.  scratch: 4096 doubles.  2 <= m <= 262144. */
LFPS_API int lfps_stage_thresholds(const double* ver, const double* sla, int32_t m, double scale,
                                   double a, int32_t materialize, double* out, double* scratch,
                                   void* stream);
/* Candidate stages (candidates.py:45-100) with thresholds thr[6] laid out
 * as above: mode 0 select_initial (in_idx unused), 1 expand (in_idx = C0,
 * offsets[n_off]), 2 finalize_probe_set (in_idx = C1; n, sink, window).
 * out_idx: capacity m (modes 0, 1) or n (mode 2); *out_count on device. */
LFPS_API int lfps_stage_candidates(int32_t mode, const double* ver, const double* sla, int32_t m,
                                   double scale, const double* thr, const int64_t* in_idx,
                                   int32_t n_in, const int32_t* offsets, int32_t n_off,
                                   int64_t base_index, int32_t n, int32_t sink, int32_t window,
                                   int64_t* out_idx, int32_t* out_count, void* stream);
/* topk_from_scores (attention.py:34-47): Top-k of (idx ascending, scores)
 * with lower-index ties; all of idx when k >= p. */
LFPS_API int lfps_stage_topk(const int64_t* idx, const double* scores, int32_t p, int32_t k,
                             int64_t* out_idx, int32_t* out_count, void* stream);
/* attention_output (attention.py:66-85) over the rows idx[nidx] (sorted;
 * NULL = all rows 0 .. nidx-1, full_attention_oracle :88-97): out[d] and
 * the softmax weights[nidx]. */
LFPS_API int lfps_stage_attend(const double* keys, const double* values, int32_t d,
                               const int64_t* idx, int32_t nidx, const double* q, double* out,
                               double* weights, int32_t* err, void* stream);
/* ScoreTablePair.update (tables.py:144-200) after the host's checks (sum of
 * weights, index range): renorm != 0 multiplies by rf first; then the slash
 * shift (slot base - 1 zeroed) and the residual fold at sel (logical) with
 * the new lazy scale `scale`; *clamps = entries clamped.  tmp: k doubles. */
LFPS_API int lfps_stage_update(double* ver, double* sla, int32_t base, int32_t m,
                               const int64_t* sel, const double* weights, int32_t k,
                               int32_t renorm, double rf, double scale, int64_t* clamps,
                               double* tmp, void* stream);
/* ScoreTablePair.grow (tables.py:202-220). */
LFPS_API int lfps_stage_grow(double* ver, double* sla, int32_t base, int32_t m, int32_t carry,
                             void* stream);
/* init_tables (tables.py:247-281): w [s, m] -> ver[m], sla[m] (logical). */
LFPS_API int lfps_stage_init_tables(const double* w, int32_t s, int32_t m, double r, double* ver,
                                    double* sla, void* stream);
/* compute_head_stats (gate.py:51-74): mean_key[d], mean_value[d], *sigma;
 * tmp: n doubles. */
LFPS_API int lfps_stage_head_stats(const double* keys, const double* values, int32_t n, int32_t d,
                                   int32_t sink, const double* q, double* mean_key,
                                   double* mean_value, double* sigma, double* tmp, int32_t* err,
                                   void* stream);
/* gate_logits + sparsity_from_logits + bypass_output (gate.py:77-147):
 * out = [sink logits S | local logits L | gexp | w_sink | w_global |
 * w_local | rho | bypass output d]. */
LFPS_API int lfps_stage_gate(const double* keys, const double* values, int32_t n, int32_t d,
                             int32_t sink, int32_t window, const double* q,
                             const double* mean_key, const double* mean_value, double sigma,
                             int32_t bypass_mode, double* out, int32_t* err, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LFPS_B200_H */
