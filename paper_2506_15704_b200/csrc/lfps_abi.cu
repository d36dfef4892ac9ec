// lfps_abi.cu -- extern "C" entry points of liblfps_b200.so (include/lfps_b200.h).
//
// Host-side validation mirrors the reference's preconditions
// (engine.py:111-120, gate.py:89-90, tables.py:303-304, config.py:44-66) and
// runs before any launch; the launch sequence of one decode step follows
// Algorithm 1 (engine.py:97-201).
#include <cstdio>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <algorithm>
#include <atomic>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(LFPS_E_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

}  // namespace

// error reporting for the other host-side translation units (kv_pool.cu)
int lfps_abi_fail(int code, const char* msg) { return fail(code, "%s", msg); }
int lfps_check_dims(const lfps_dims* d);

namespace {

constexpr int kMaxMcap = 510 * 512;     // slash table <= 1022 blocks (32 dirty words)
constexpr int kMaxM = kMaxMcap - 2;     // k_select.cu: a window spans <= 512 blocks

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

int check_dims(const lfps_dims* d) {
  if (!d) return fail(LFPS_E_INVALID, "dims is NULL");
  if (d->batch < 1 || d->kv_heads < 1) return fail(LFPS_E_INVALID, "batch and kv_heads must be >= 1");
  if (!(d->group == 1 || d->group == 2 || d->group == 4 || d->group == 8))
    return fail(LFPS_E_UNSUPPORTED, "group (q heads per KV head) must be 1, 2, 4 or 8, got %d", d->group);
  if (!(d->d == 32 || d->d == 64 || d->d == 128 || d->d == 256))
    return fail(LFPS_E_UNSUPPORTED, "head dimension must be 32, 64, 128 or 256, got %d", d->d);
  if (d->m_cap < 2 || (d->m_cap & 1)) return fail(LFPS_E_INVALID, "m_cap must be even and >= 2");
  if (d->m_cap > kMaxMcap)
    return fail(LFPS_E_UNSUPPORTED, "m_cap must be <= %d", kMaxMcap);
  if (d->n_max < 2) return fail(LFPS_E_INVALID, "n_max must be >= 2");
  if ((long long)d->batch * d->kv_heads * d->group * 2 > 65535)
    return fail(LFPS_E_UNSUPPORTED, "too many sessions for one launch (B*Hq <= 32767)");
  return LFPS_OK;
}

int check_params(const lfps_params* p, const lfps_dims* d) {
  if (!p) return fail(LFPS_E_INVALID, "params is NULL");
  if (!(p->r >= 0.0 && p->r < 1.0)) return fail(LFPS_E_INVALID, "r must be in [0, 1), got %g", p->r);
  if (!(p->epsilon > 0.0 && p->epsilon <= 1.0))
    return fail(LFPS_E_INVALID, "epsilon must be in (0, 1], got %g", p->epsilon);
  if (!(p->a > 0.0)) return fail(LFPS_E_INVALID, "a must be > 0, got %g", p->a);
  if (!(p->k_fraction > 0.0 && p->k_fraction <= 1.0))
    return fail(LFPS_E_INVALID, "k_fraction must be in (0, 1], got %g", p->k_fraction);
  if (p->s < 1) return fail(LFPS_E_INVALID, "s must be >= 1");
  if (p->sink_count < 1 || p->sink_count > 31)
    return fail(LFPS_E_UNSUPPORTED, "sink_count must be in [1, 31], got %d", p->sink_count);
  if (p->local_window < 1 || p->local_window > 64)
    return fail(LFPS_E_UNSUPPORTED, "local_window must be in [1, 64], got %d", p->local_window);
  if (p->bypass_mode != 0 && p->bypass_mode != 1) return fail(LFPS_E_INVALID, "bad bypass_mode");
  if (p->n_offsets < 1 || p->n_offsets > 16) return fail(LFPS_E_UNSUPPORTED, "1..16 offsets supported");
  bool zero = false;
  for (int i = 0; i < p->n_offsets; ++i) {
    if (p->offsets[i] < -31 || p->offsets[i] > 31)
      return fail(LFPS_E_UNSUPPORTED, "expansion offsets must lie in [-31, 31]");
    zero |= p->offsets[i] == 0;
  }
  if (!zero) return fail(LFPS_E_INVALID, "expansion_offsets must contain 0");
  if (std::fabs(p->sqrt_d - std::sqrt((double)d->d)) > 0.0)
    return fail(LFPS_E_INVALID, "sqrt_d must equal sqrt(d)");
  return LFPS_OK;
}

// slash table: 2 * roundup(m_cap, 512) + 1024 slots; the window starts out
// ending at the home slot roundup(m_cap, 512) + 512 and can grow m_cap slots
// down (slash shifts) and m_cap slots up (gated steps) without wrapping
int slash_home(int m_cap) { return (m_cap + lfps::kBlk - 1) / lfps::kBlk * lfps::kBlk + lfps::kBlk; }
int slash_cap(int m_cap) { return 2 * slash_home(m_cap); }

int layout(const lfps_dims* d, lfps_ws_layout* L) {
  const size_t NS = (size_t)d->batch * d->kv_heads * d->group;
  const size_t NI = 2 * NS;
  // per-session lists: m_cap entries rounded up to 32 (128-byte aligned rows,
  // so every session's score list takes the vector loads of k_topk.cu)
  const size_t cap = align_up((size_t)d->m_cap, 32);
  memset(L, 0, sizeof(*L));
  L->list_cap = (int)cap;
  L->words = (int)((cap + 511) / 512 * 16);   // whole 512-slot chunks
  L->nblk = slash_cap(d->m_cap) / lfps::kBlk;
  L->dirty_words = (L->nblk + 31) / 32;
  size_t o = 0;
  auto take = [&](size_t bytes) { const size_t at = o; o = align_up(o + bytes, 256); return at; };
  L->rho = take(NS * 8);
  L->bypass = take(NS * 4);
  L->err = take((NS + 1) * 4);
  L->out = take(NS * d->d * 4);
  L->thr = take(NS * 8 * 8);
  L->counts = take(NS * lfps::CNT_N * 4);
  L->bits = take(NI * (size_t)L->words * 4);
  L->probe_idx = take(NS * cap * 4);
  L->probe_score = take(NS * cap * 4);
  L->c2_idx = take(NS * cap * 4);
  L->c2_score = take(NS * cap * 4);
  L->uw = take(NS * cap * 8);
  // bootstrap scratch (f64 logits) aliases probe_idx + probe_score
  L->scratch = L->probe_idx;
  L->bsum = take(NI * (size_t)L->nblk * 4 * 8);
  L->bmax = take(NI * (size_t)L->nblk * 8);
  L->dirty = take(NI * (size_t)L->dirty_words * 4);
  L->valid = take(NS * 4);
  L->wstat = take(NS * 2 * 8);
  L->trace = take(NS * 16 * 8);
  L->done = take(64);
  L->hot = take(NI * (size_t)(16 * L->nblk + 1) * 8);
  L->thr_next = take(NS * 8 * 8);
  L->total_bytes = o;
  return LFPS_OK;
}

// the error stamp of every call other than a decode step (bootstrap, exact
// path); decode steps draw distinct stamps from next_epoch()
constexpr int kOtherStamp = 0x7ffffff;

int make_ctx(const lfps_dims* d, const lfps_params* p, const lfps_state* st,
             const lfps_workspace* ws, lfps::Ctx* c) {
  int rc = check_dims(d);
  if (rc) return rc;
  rc = check_params(p, d);
  if (rc) return rc;
  if (!st || !ws || !ws->base) return fail(LFPS_E_INVALID, "state/workspace is NULL");
  lfps_ws_layout L;
  layout(d, &L);
  if (ws->bytes < L.total_bytes)
    return fail(LFPS_E_INVALID, "workspace too small: %zu < %zu bytes", ws->bytes, L.total_bytes);
  memset(c, 0, sizeof(*c));
  c->B = d->batch; c->Hkv = d->kv_heads; c->G = d->group; c->Hq = d->kv_heads * d->group;
  c->NS = c->B * c->Hq; c->s_off = 0; c->s_cnt = c->NS; c->epoch = kOtherStamp; c->d = d->d; c->n_max = d->n_max; c->m_cap = d->m_cap;
  c->sla_cap = slash_cap(d->m_cap); c->sla_home = slash_home(d->m_cap);
  c->words = L.words; c->list_cap = L.list_cap;
  c->r = p->r; c->eps = p->epsilon; c->a = p->a; c->frac = p->k_fraction; c->sqrt_d = p->sqrt_d;
  c->sqrt_d_f32 = p->sqrt_d_f32; c->s = p->s; c->S = p->sink_count; c->L = p->local_window;
  c->bypass_mode = p->bypass_mode; c->exhaustive = p->exhaustive; c->n_off = p->n_offsets;
  c->flags = p->flags;
  for (int i = 0; i < 16; ++i) c->off[i] = i < p->n_offsets ? p->offsets[i] : 0;
  c->K = static_cast<const __nv_bfloat16*>(st->k_cache);
  c->V = static_cast<const __nv_bfloat16*>(st->v_cache);
  c->Kw = static_cast<__nv_bfloat16*>(st->k_cache);
  c->Vw = static_cast<__nv_bfloat16*>(st->v_cache);
  c->n_ctx = st->n_ctx; c->ver = st->ver; c->sla = st->sla; c->scale = st->scale;
  c->sla_base = st->sla_base; c->clamp_count = reinterpret_cast<long long*>(st->clamp_count);
  c->mean_key = st->mean_key; c->mean_value = st->mean_value; c->sigma = st->sigma_hat_sq;
  if (!c->K || !c->V || !c->n_ctx || !c->ver || !c->sla || !c->scale || !c->sla_base ||
      !c->clamp_count || !c->mean_key || !c->mean_value || !c->sigma)
    return fail(LFPS_E_INVALID, "a state pointer is NULL");
  c->bt = st->block_table;
  c->bs_shift = 31;
  c->bs_mask = 0x7fffffff;
  c->max_blocks = 0;
  if (st->block_table) {
    const int br = st->block_rows;
    if (br < 1 || br > (1 << 16) || (br & (br - 1)))
      return fail(LFPS_E_INVALID, "block_rows must be a power of two in [1, 65536], got %d", br);
    if (st->max_blocks < 1 || (long long)st->max_blocks * br != d->n_max)
      return fail(LFPS_E_INVALID, "block table: n_max (%d) must equal max_blocks (%d) * block_rows (%d)",
                  d->n_max, st->max_blocks, br);
    c->bs_shift = __builtin_ctz((unsigned)br);
    c->bs_mask = br - 1;
    c->max_blocks = st->max_blocks;
  }
  char* base = static_cast<char*>(ws->base);
  c->rho = reinterpret_cast<double*>(base + L.rho);
  c->bypass = reinterpret_cast<int*>(base + L.bypass);
  c->err = reinterpret_cast<int*>(base + L.err);
  c->out = reinterpret_cast<float*>(base + L.out);
  c->thr = reinterpret_cast<double*>(base + L.thr);
  c->counts = reinterpret_cast<int*>(base + L.counts);
  c->bits = reinterpret_cast<uint32_t*>(base + L.bits);
  c->probe_idx = reinterpret_cast<int*>(base + L.probe_idx);
  c->probe_score = reinterpret_cast<float*>(base + L.probe_score);
  c->c2_idx = reinterpret_cast<int*>(base + L.c2_idx);
  c->c2_score = reinterpret_cast<float*>(base + L.c2_score);
  c->uw = reinterpret_cast<double*>(base + L.uw);
  c->scratch = reinterpret_cast<double*>(base + L.scratch);
  c->bw.bsum = reinterpret_cast<double*>(base + L.bsum);
  c->bw.bmax = reinterpret_cast<double*>(base + L.bmax);
  c->bw.dirty = reinterpret_cast<uint32_t*>(base + L.dirty);
  c->bw.valid = reinterpret_cast<int*>(base + L.valid);
  c->bw.wstat = reinterpret_cast<double*>(base + L.wstat);
  c->trace = reinterpret_cast<long long*>(base + L.trace);
  c->done = reinterpret_cast<unsigned*>(base + L.done);
  c->hot = reinterpret_cast<int2*>(base + L.hot);
  c->thr_next = reinterpret_cast<double*>(base + L.thr_next);
  c->bw.nblk = L.nblk;
  c->bw.dwords = L.dirty_words;
  return LFPS_OK;
}

// decode preconditions on the host copy of n (engine.py:114-120, gate.py:89-90)
int check_context(const lfps::Ctx& c, const int32_t* n_host, bool append, int* m_max) {
  if (!n_host) return fail(LFPS_E_INVALID, "n_host is NULL");
  int mm = 0;
  for (int b = 0; b < c.B; ++b) {
    const int n = n_host[b];
    if (n <= c.S + c.L)
      return fail(LFPS_E_INVALID, "request %d: context %d shorter than sink_count + local_window", b, n);
    const int m = n - c.S;
    if (append && n >= c.n_max)
      return fail(LFPS_E_INVALID, "request %d: KV cache full (n=%d, n_max=%d)", b, n, c.n_max);
    if (m + 2 > c.m_cap)
      return fail(LFPS_E_INVALID, "request %d: tables full (m=%d, m_cap=%d)", b, m, c.m_cap);
    if (m > kMaxM) return fail(LFPS_E_UNSUPPORTED, "context %d exceeds the scan limit", n);
    if (m > mm) mm = m;
  }
  *m_max = mm;
  return LFPS_OK;
}

#define LAUNCH(x)                                         \
  do {                                                    \
    cudaError_t e_ = (x);                                 \
    if (e_ != cudaSuccess) return cuda_fail(e_, #x);      \
  } while (0)

// ---- optional per-kernel CUDA-event timing (lfps_profile_*) ----------------
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t prof_event() {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

// launch `x` on stream `sm`, bracketed by events when profiling is on
#define LAUNCH_P(name, sm, x)                                      \
  do {                                                             \
    cudaEvent_t a_ = nullptr;                                      \
    if (g_prof_on) {                                               \
      a_ = prof_event();                                           \
      cudaEventRecord(a_, sm);                                     \
    }                                                              \
    LAUNCH(x);                                                     \
    if (g_prof_on) {                                               \
      cudaEvent_t b_ = prof_event();                               \
      cudaEventRecord(b_, sm);                                     \
      std::lock_guard<std::mutex> g_(g_prof_mu);                   \
      g_prof.push_back({name, a_, b_});                            \
    }                                                              \
  } while (0)

// ---- internal streams for session-group concurrency (LFPS_FLAG_SPLIT) -------
// call stamps for err[0] (Ctx::epoch): a decode step that fails leaves its
// stamp in err[0]; the next step's kernels compare against their own stamp,
// so no clearing kernel is needed (per-session codes are cleared by the gate)
std::atomic<int> g_epoch{1};
int next_epoch() {
  int e = g_epoch.fetch_add(1) & 0x3ffffff;          // < 2^26; graph steps draw [2^26, 2^27)
  return (e && e != kOtherStamp) ? e : next_epoch();
}

#ifndef LFPS_SPLIT_GROUPS
#define LFPS_SPLIT_GROUPS 4
#endif
constexpr int kSplitGroups = LFPS_SPLIT_GROUPS;   // session groups of LFPS_FLAG_SPLIT
#ifndef LFPS_SPLIT_MIN
#define LFPS_SPLIT_MIN 1024
#endif
constexpr int kSplitMin = LFPS_SPLIT_MIN;         // sessions below which the split is off
#ifndef LFPS_SELECT_AHEAD
#define LFPS_SELECT_AHEAD 1
#endif
constexpr bool kSelectAhead = LFPS_SELECT_AHEAD != 0;   // select beside the gate, not after it
#ifndef LFPS_AHEAD_SPLIT
#define LFPS_AHEAD_SPLIT 0       // select beside the gate in split steps too
#endif
#ifndef LFPS_GATE_SIDE
#define LFPS_GATE_SIDE 1
#endif
constexpr bool kGateSide = LFPS_GATE_SIDE != 0;   // the gate on the side stream (with select ahead)
// Internal streams and events of one workspace (one BatchedSession): the
// fork/join events of a step are re-recorded by every call, so they must not
// be shared between sessions that different host threads step concurrently
// (cudaStreamWaitEvent binds to the event's latest record at the time of the
// call).  Pipes are created on a workspace's first decode step, keyed by
// (device, workspace base), and destroyed by lfps_workspace_release.
struct Pipe {
  std::mutex mu;                            // one enqueue sequence at a time
  cudaStream_t st[kSplitGroups] = {};
  cudaStream_t aux[kSplitGroups] = {};      // the stats kernel, concurrent with the gate
  cudaEvent_t fork = nullptr, join[kSplitGroups] = {}, stats[kSplitGroups] = {};
  cudaStream_t copy = nullptr;              // host output copy beside the commit
  cudaEvent_t out_ready = nullptr, out_done = nullptr;
  cudaEvent_t out_ext = nullptr;            // the output copy's completion for the host
                                            // (recorded as an external event node in graphs)
  cudaStream_t in = nullptr;                // host input copy beside the stats kernel
  cudaEvent_t in_ready = nullptr;
  cudaStream_t cap = nullptr;               // CUDA-graph capture of a decode step
  std::vector<struct StepGraph*> graphs;    // captured steps, most recent last
  void* stage = nullptr;                    // graph steps with device inputs: the
  size_t stage_bytes = 0;                   // inputs are copied here first
  int pre_epoch = 0;                        // lfps_decode_prefetch's call stamp, until the
                                            // LFPS_FLAG_PREFETCHED step that consumes it
};
std::mutex g_pipe_mu;

// A decode step captured as a CUDA graph (see decode_impl): everything a
// replay cannot change is in the key; the host buffers of the input and
// output copies are set per replay on their memcpy nodes.
struct GraphKey {
  lfps_dims dims;
  lfps_params params;
  lfps_state state;
  const void* ws;
  const void *q, *k_new, *v_new;
  int m_bucket, has_in, has_out;
  bool operator==(const GraphKey& o) const { return memcmp(this, &o, sizeof(*this)) == 0; }
};
struct StepGraph {
  GraphKey key;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphNode_t in_node = nullptr, out_node = nullptr;
  const void* in_host = nullptr;
  void* out_host = nullptr;
  size_t in_bytes = 0, out_bytes = 0;
  ~StepGraph() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
  }
};
constexpr int kMaxGraphs = 4;
std::map<std::pair<int, const void*>, std::unique_ptr<Pipe>> g_pipes;

void destroy_pipe(Pipe& p) {
  for (StepGraph* g : p.graphs) delete g;
  p.graphs.clear();
  if (p.stage) cudaFree(p.stage);
  if (p.cap) cudaStreamDestroy(p.cap);
  for (cudaStream_t* sp : {&p.st[0], &p.st[kSplitGroups - 1], &p.aux[0], &p.aux[kSplitGroups - 1],
                           &p.copy, &p.in})
    if (*sp) cudaStreamSynchronize(*sp);
  for (int i = 0; i < kSplitGroups; ++i) {
    if (p.st[i]) cudaStreamDestroy(p.st[i]);
    if (p.aux[i]) cudaStreamDestroy(p.aux[i]);
    if (p.join[i]) cudaEventDestroy(p.join[i]);
    if (p.stats[i]) cudaEventDestroy(p.stats[i]);
  }
  for (cudaEvent_t ev : {p.fork, p.out_ready, p.out_done, p.out_ext, p.in_ready})
    if (ev) cudaEventDestroy(ev);
  if (p.copy) cudaStreamDestroy(p.copy);
  if (p.in) cudaStreamDestroy(p.in);
}

cudaError_t create_pipe(Pipe& p) {
  cudaError_t e;
  for (int i = 0; i < kSplitGroups; ++i) {
    if ((e = cudaStreamCreateWithFlags(&p.st[i], cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaStreamCreateWithFlags(&p.aux[i], cudaStreamNonBlocking)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&p.join[i], cudaEventDisableTiming)) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&p.stats[i], cudaEventDisableTiming)) != cudaSuccess) return e;
  }
  if ((e = cudaEventCreateWithFlags(&p.fork, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&p.copy, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaEventCreateWithFlags(&p.out_ready, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaEventCreateWithFlags(&p.out_done, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaEventCreateWithFlags(&p.out_ext, cudaEventDisableTiming)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&p.in, cudaStreamNonBlocking)) != cudaSuccess) return e;
  if ((e = cudaStreamCreateWithFlags(&p.cap, cudaStreamNonBlocking)) != cudaSuccess) return e;
  return cudaEventCreateWithFlags(&p.in_ready, cudaEventDisableTiming);
}

cudaError_t get_pipe(const void* ws_base, Pipe** out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> g(g_pipe_mu);
  std::unique_ptr<Pipe>& p = g_pipes[{dev, ws_base}];
  if (!p) {
    std::unique_ptr<Pipe> np(new Pipe());
    if ((e = create_pipe(*np)) != cudaSuccess) {
      destroy_pipe(*np);
      g_pipes.erase({dev, ws_base});
      return e;
    }
    p = std::move(np);
  }
  *out = p.get();
  return cudaSuccess;
}

}  // namespace

extern "C" {

int lfps_abi_version(void) { return LFPS_ABI_VERSION; }

int lfps_wait_output(const lfps_workspace* ws) {
  if (!ws || !ws->base) return fail(LFPS_E_INVALID, "workspace is NULL");
  Pipe* pp = nullptr;
  {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    std::lock_guard<std::mutex> g(g_pipe_mu);
    auto it = g_pipes.find({dev, ws->base});
    if (it == g_pipes.end()) return fail(LFPS_E_INVALID, "no decode step on this workspace yet");
    pp = it->second.get();
  }
  // the last host-output step's copy (its event is re-recorded by every such
  // step, in CUDA-graph replays too)
  cudaError_t e = cudaEventSynchronize(pp->out_ext);
  return e == cudaSuccess ? LFPS_OK : cuda_fail(e, "cudaEventSynchronize");
}

const char* lfps_last_error(void) { return g_err; }

int lfps_workspace_layout(const lfps_dims* dims, lfps_ws_layout* out) {
  int rc = check_dims(dims);
  if (rc) return rc;
  if (!out) return fail(LFPS_E_INVALID, "out is NULL");
  return layout(dims, out);
}

// clear, gate, select, finish, update (with append and commit); with
// LFPS_FLAG_SPLIT (and >= 256 sessions) gate/select/finish run per half
int lfps_decode_launches(const lfps_dims* dims, int32_t flags) {
  // per group: gate | stats, select, finish (LFPS_FLAG_PREFETCHED: gate,
  // finish -- stats and select ran in lfps_decode_prefetch), then the update
  const long long ns = dims ? (long long)dims->batch * dims->kv_heads * dims->group : 0;
  const int per = (flags & LFPS_FLAG_PREFETCHED) ? 2 : 4;
  if (dims && (flags & LFPS_FLAG_SPLIT) && ns >= kSplitMin) return 1 + per * kSplitGroups;
  return 1 + per;
}

int lfps_workspace_release(const lfps_workspace* ws) {
  if (!ws || !ws->base) return fail(LFPS_E_INVALID, "workspace is NULL");
  std::unique_ptr<Pipe> gone;
  {
    std::lock_guard<std::mutex> g(g_pipe_mu);
    for (auto it = g_pipes.begin(); it != g_pipes.end(); ++it)
      if (it->first.second == ws->base) {
        gone = std::move(it->second);
        g_pipes.erase(it);
        break;
      }
  }
  if (gone) {
    std::lock_guard<std::mutex> g(gone->mu);
    destroy_pipe(*gone);
  }
  return LFPS_OK;
}

int lfps_slash_capacity(const lfps_dims* dims) {
  int rc = check_dims(dims);
  if (rc) return rc;
  return slash_cap(dims->m_cap);
}

int lfps_profile_enable(int on) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = on != 0;
  return LFPS_OK;
}

int lfps_profile_collect(lfps_kernel_time* out, int32_t cap, int32_t* n_out) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!out || !n_out || cap < 1) return fail(LFPS_E_INVALID, "bad profile buffer");
  int n = 0;
  for (const ProfRec& r : g_prof) {
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    int k = 0;
    while (k < n && strncmp(out[k].name, r.name, sizeof(out[k].name)) != 0) ++k;
    if (k == n) {
      if (n == cap) continue;
      memset(&out[n], 0, sizeof(out[n]));
      strncpy(out[n].name, r.name, sizeof(out[n].name) - 1);
      ++n;
    }
    out[k].launches += 1;
    out[k].total_ms += ms;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_prof.clear();
  *n_out = n;
  return LFPS_OK;
}
int lfps_exact_launches(void) { return 4; }

int lfps_bootstrap_tables(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                          const lfps_workspace* ws, const float* weights, int32_t s_begin,
                          int32_t count, int32_t m0, void* stream) {
  lfps::Ctx c;
  int rc = make_ctx(dims, p, st, ws, &c);
  if (rc) return rc;
  if (!weights) return fail(LFPS_E_INVALID, "weights is NULL");
  if (s_begin < 0 || count < 1 || s_begin + count > c.NS)
    return fail(LFPS_E_INVALID, "session range [%d, %d) outside [0, %d)", s_begin, s_begin + count, c.NS);
  if (m0 < 1) return fail(LFPS_E_INVALID, "prefill weight vectors are empty");
  if (m0 + 2 > c.m_cap) return fail(LFPS_E_INVALID, "m0=%d does not fit m_cap=%d", m0, c.m_cap);
  if (count > 65535 || c.s > 65535) return fail(LFPS_E_UNSUPPORTED, "too many sessions per call");
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  LAUNCH(lfps::launch_boot_tables(c, weights, s_begin, count, m0, sm));
  return LFPS_OK;
}

int lfps_bootstrap_stats(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                         const lfps_workspace* ws, const void* last_query, void* stream) {
  lfps::Ctx c;
  int rc = make_ctx(dims, p, st, ws, &c);
  if (rc) return rc;
  if (!last_query) return fail(LFPS_E_INVALID, "last_query is NULL");
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  LAUNCH(lfps::launch_boot_stats(c, static_cast<const __nv_bfloat16*>(last_query), c.m_cap, 0, c.B,
                                 sm));
  return LFPS_OK;
}

int lfps_bootstrap_stats_requests(const lfps_dims* dims, const lfps_params* p,
                                  const lfps_state* st, const lfps_workspace* ws,
                                  const void* last_query, int32_t b_begin, int32_t b_count,
                                  void* stream) {
  lfps::Ctx c;
  int rc = make_ctx(dims, p, st, ws, &c);
  if (rc) return rc;
  if (!last_query) return fail(LFPS_E_INVALID, "last_query is NULL");
  if (b_begin < 0 || b_count < 1 || b_begin + b_count > c.B)
    return fail(LFPS_E_INVALID, "request range [%d, %d) outside [0, %d)", b_begin, b_begin + b_count, c.B);
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  LAUNCH(lfps::launch_boot_stats(c, static_cast<const __nv_bfloat16*>(last_query), c.m_cap, b_begin,
                                 b_count, sm));
  return LFPS_OK;
}

static int decode_impl(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                       const lfps_workspace* ws, const void* q, const void* k_new,
                       const void* v_new, const int32_t* n_host, void* out_host,
                       const void* in_host, void* stream);

int lfps_decode_prefetch(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                         const lfps_workspace* ws, const int32_t* n_host, void* stream) {
  lfps::Ctx c;
  int rc = make_ctx(dims, p, st, ws, &c);
  if (rc) return rc;
  int m_max = 0;
  rc = check_context(c, n_host, true, &m_max);
  if (rc) return rc;
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  Pipe* pp = nullptr;
  LAUNCH(get_pipe(ws->base, &pp));
  std::lock_guard<std::mutex> pipe_lock(pp->mu);
  c.epoch = next_epoch();
  c.prefetch = 1;
  // thresholds + C0 words of every (session, table), then C + D of every
  // session, on the caller's stream (no gate: nothing here reads q)
  LAUNCH_P("stats", sm, lfps::launch_stats(c, sm));
  LAUNCH_P("select", sm, lfps::launch_select(c, m_max, sm));
  pp->pre_epoch = c.epoch;
  return LFPS_OK;
}

int lfps_decode_step(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                     const lfps_workspace* ws, const void* q, const void* k_new,
                     const void* v_new, const int32_t* n_host, void* stream) {
  return decode_impl(dims, p, st, ws, q, k_new, v_new, n_host, nullptr, nullptr, stream);
}

int lfps_decode_step_host_out(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                              const lfps_workspace* ws, const void* q, const void* k_new,
                              const void* v_new, const int32_t* n_host, void* out_host,
                              void* stream) {
  if (!out_host) return fail(LFPS_E_INVALID, "out_host is NULL");
  return decode_impl(dims, p, st, ws, q, k_new, v_new, n_host, out_host, nullptr, stream);
}

int64_t lfps_step_input_bytes(const lfps_dims* dims) {
  if (check_dims(dims)) return LFPS_E_INVALID;
  const int64_t units = (int64_t)dims->batch * dims->kv_heads;
  return (units * dims->group + 2 * units) * dims->d * 2;
}

int lfps_decode_step_host_io(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                             const lfps_workspace* ws, const void* in_host, void* in_dev,
                             const int32_t* n_host, void* out_host, void* stream) {
  int rc = check_dims(dims);
  if (rc) return rc;
  if (!in_host || !in_dev) return fail(LFPS_E_INVALID, "in_host/in_dev is NULL");
  const size_t units = (size_t)dims->batch * dims->kv_heads;
  const __nv_bfloat16* q = static_cast<const __nv_bfloat16*>(in_dev);
  const __nv_bfloat16* k_new = q + units * dims->group * dims->d;
  const __nv_bfloat16* v_new = k_new + units * dims->d;
  return decode_impl(dims, p, st, ws, q, k_new, v_new, n_host, out_host, in_host, stream);
}

// Enqueue one decode step on stream sm (the caller's, or the capture stream).
// Stats and select do not depend on the gate (they serve every session, and
// the finish treats gated sessions and kappa = 0 as after a prefetch), so
// the gate runs on an internal stream forked from sm and stats -> select ->
// finish stay one PDL chain on sm, the finish joining the gate.  (Select
// after the gate, LFPS_SELECT_AHEAD=0, measured the same on the device and
// 10 us slower end to end at C1/C2: the gate waits for the input copy.)
// LFPS_FLAG_SPLIT (>= kSplitMin sessions) instead runs kSplitGroups session
// groups, each [gate | stats] -> select -> finish, on their own streams
// (stats on an internal stream, joined before select); the update (commit)
// joins them on sm.  Under lfps_profile_enable
// everything runs serially on sm so each kernel is timed alone.  Host
// inputs (lfps_decode_step_host_io): q | k_new | v_new are contiguous from q
// on; the copy starts with the step on its own stream (after the caller's
// previous work, which may still read the buffer) and only the gate waits
// for it -- the stats kernel does not read the inputs.  A graph step
// (c.stamp set) starts with the kernel that draws its call stamp.
static int enqueue_step(const lfps::Ctx& c, Pipe* pp, cudaStream_t sm, const void* q,
                        const void* k_new, const void* v_new, void* out_host,
                        const void* in_host, int m_max) {
  const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(q);
  const size_t in_bytes = ((size_t)c.NS + 2 * (size_t)c.B * c.Hkv) * c.d * sizeof(__nv_bfloat16);
  if (c.stamp) LAUNCH(lfps::launch_step_begin(c, sm));
  if (in_host && g_prof_on)
    LAUNCH(cudaMemcpyAsync(const_cast<void*>(q), in_host, in_bytes, cudaMemcpyHostToDevice, sm));
  const bool pre = (c.flags & LFPS_FLAG_PREFETCHED) != 0;   // stats + select already ran
  // select beside the gate: unsplit steps only (with the split groups the
  // finish's cross-stream join on the gate costs more than it hides)
  const bool split = (c.flags & LFPS_FLAG_SPLIT) && !g_prof_on && c.NS >= kSplitMin;
  const bool ahead = !pre && kSelectAhead &&
                     (LFPS_AHEAD_SPLIT || !((c.flags & LFPS_FLAG_SPLIT) && c.NS >= kSplitMin));
  if (g_prof_on) {
    lfps::Ctx cf = c;
    cf.prefetch = ahead;
    LAUNCH_P("gate", sm, lfps::launch_gate(c, qb, sm));
    if (!pre) {
      LAUNCH_P("stats", sm, lfps::launch_stats(cf, sm));
      LAUNCH_P("select", sm, lfps::launch_select(cf, m_max, sm));
    }
  } else {
    LAUNCH(cudaEventRecord(pp->fork, sm));
    if (in_host) {
      LAUNCH(cudaStreamWaitEvent(pp->in, pp->fork, 0));
      LAUNCH(cudaMemcpyAsync(const_cast<void*>(q), in_host, in_bytes, cudaMemcpyHostToDevice, pp->in));
      LAUNCH(cudaEventRecord(pp->in_ready, pp->in));
    }
  }
  const int groups = split ? kSplitGroups : 1;
  const int per = (c.NS / groups + 31) / 32 * 32;
  for (int g = 0; g < groups; ++g) {
    lfps::Ctx cg = c;
    cg.s_off = g * per;
    cg.s_cnt = g == groups - 1 ? c.NS - g * per : per;
    if (ahead) cg.prefetch = 1;
    cudaStream_t gs = split ? pp->st[g] : sm;
    if (!g_prof_on) {
      cudaStream_t as = pp->aux[g];
      if (split) LAUNCH(cudaStreamWaitEvent(gs, pp->fork, 0));
      if (ahead && kGateSide) {
        // the gate (after the input copy) on the side stream; stats ->
        // select -> finish stay one programmatic-launch chain on the group's
        LAUNCH(cudaStreamWaitEvent(as, pp->fork, 0));
        if (in_host) LAUNCH(cudaStreamWaitEvent(as, pp->in_ready, 0));
        LAUNCH(lfps::launch_gate(cg, qb, as));
        LAUNCH(cudaEventRecord(pp->stats[g], as));
        LAUNCH(lfps::launch_stats(cg, gs));
        LAUNCH(lfps::launch_select(cg, m_max, gs));
        LAUNCH(cudaStreamWaitEvent(gs, pp->stats[g], 0));
      } else if (ahead) {
        // the sets are built beside the gate (and the input copy): select
        // follows stats on the side stream, the finish joins both
        LAUNCH(cudaStreamWaitEvent(as, pp->fork, 0));
        LAUNCH(lfps::launch_stats(cg, as));
        LAUNCH(lfps::launch_select(cg, m_max, as));
        LAUNCH(cudaEventRecord(pp->stats[g], as));
      } else if (!pre) {
        LAUNCH(cudaStreamWaitEvent(as, pp->fork, 0));
        LAUNCH(lfps::launch_stats(cg, as));
        LAUNCH(cudaEventRecord(pp->stats[g], as));
      }
      if (!(ahead && kGateSide)) {
        if (in_host) LAUNCH(cudaStreamWaitEvent(gs, pp->in_ready, 0));
        LAUNCH(lfps::launch_gate(cg, qb, gs));
      }
      if (ahead) {
        if (!kGateSide) LAUNCH(cudaStreamWaitEvent(gs, pp->stats[g], 0));
      } else if (!pre) {
        LAUNCH(cudaStreamWaitEvent(gs, pp->stats[g], 0));
        LAUNCH(lfps::launch_select(cg, m_max, gs));
      }
    }
    LAUNCH_P("finish", gs, lfps::launch_finish(cg, qb, gs));
    if (split) {
      LAUNCH(cudaEventRecord(pp->join[g], gs));
      LAUNCH(cudaStreamWaitEvent(sm, pp->join[g], 0));
    }
  }
  // the output is final here (gate + finish); the commit does not touch it
  if (out_host) {
    LAUNCH(cudaEventRecord(pp->out_ready, sm));
    LAUNCH(cudaStreamWaitEvent(pp->copy, pp->out_ready, 0));
    LAUNCH(cudaMemcpyAsync(out_host, c.out, (size_t)c.NS * c.d * sizeof(float),
                           cudaMemcpyDeviceToHost, pp->copy));
    // (the host's event first: the join on out_done then covers its graph
    // node; under capture it is recorded as an external event node so that
    // replays record it)
    if (c.stamp) LAUNCH(cudaEventRecordWithFlags(pp->out_ext, pp->copy, cudaEventRecordExternal));
    else LAUNCH(cudaEventRecord(pp->out_ext, pp->copy));
    LAUNCH(cudaEventRecord(pp->out_done, pp->copy));
  }
  LAUNCH_P("update", sm, lfps::launch_update(c, static_cast<const __nv_bfloat16*>(k_new),
                                              static_cast<const __nv_bfloat16*>(v_new), sm));
  if (out_host) LAUNCH(cudaStreamWaitEvent(sm, pp->out_done, 0));
  return LFPS_OK;
}

// Capture a step as a CUDA graph (on the pipe's capture stream) and find its
// host-copy nodes.
static int capture_step(lfps::Ctx c, Pipe* pp, const GraphKey& key, const void* q,
                        const void* k_new, const void* v_new, void* out_host,
                        const void* in_host, int m_bucket, StepGraph** out) {
  StepGraph* g = new StepGraph();
  g->key = key;
  cudaError_t e = cudaStreamBeginCapture(pp->cap, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) { delete g; return cuda_fail(e, "cudaStreamBeginCapture"); }
  const int rc = enqueue_step(c, pp, pp->cap, q, k_new, v_new, out_host, in_host, m_bucket);
  e = cudaStreamEndCapture(pp->cap, &g->graph);
  if (rc) { delete g; return rc; }
  if (e != cudaSuccess) { delete g; return cuda_fail(e, "cudaStreamEndCapture"); }
  size_t nn = 0;
  if ((e = cudaGraphGetNodes(g->graph, nullptr, &nn)) != cudaSuccess) { delete g; return cuda_fail(e, "cudaGraphGetNodes"); }
  std::vector<cudaGraphNode_t> nodes(nn);
  if ((e = cudaGraphGetNodes(g->graph, nodes.data(), &nn)) != cudaSuccess) { delete g; return cuda_fail(e, "cudaGraphGetNodes"); }
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(nd, &t) != cudaSuccess || t != cudaGraphNodeTypeMemcpy) continue;
    cudaMemcpy3DParms mp = {};
    if (cudaGraphMemcpyNodeGetParams(nd, &mp) != cudaSuccess) continue;
    if (mp.kind == cudaMemcpyHostToDevice) g->in_node = nd;
    else if (mp.kind == cudaMemcpyDeviceToHost) g->out_node = nd;
  }
  if (const char* dot = getenv("LFPS_GRAPH_DOT"))     // diagnostics: the captured step
    cudaGraphDebugDotPrint(g->graph, dot, cudaGraphDebugDotFlagsVerbose);
  if ((e = cudaGraphInstantiate(&g->exec, g->graph, 0)) != cudaSuccess) {
    delete g;
    return cuda_fail(e, "cudaGraphInstantiate");
  }
  g->in_host = in_host;
  g->out_host = out_host;
  g->in_bytes = ((size_t)c.NS + 2 * (size_t)c.B * c.Hkv) * c.d * sizeof(__nv_bfloat16);
  g->out_bytes = (size_t)c.NS * c.d * sizeof(float);
  *out = g;
  return LFPS_OK;
}

static int decode_impl(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                       const lfps_workspace* ws, const void* q, const void* k_new,
                       const void* v_new, const int32_t* n_host, void* out_host,
                       const void* in_host, void* stream) {
  lfps::Ctx c;
  int rc = make_ctx(dims, p, st, ws, &c);
  if (rc) return rc;
  if (!q || !k_new || !v_new) return fail(LFPS_E_INVALID, "q/k_new/v_new is NULL");
  int m_max = 0;
  rc = check_context(c, n_host, true, &m_max);
  if (rc) return rc;
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  Pipe* pp = nullptr;
  LAUNCH(get_pipe(ws->base, &pp));
  std::lock_guard<std::mutex> pipe_lock(pp->mu);
  if (c.flags & LFPS_FLAG_PREFETCHED) {
    // the candidate sets come from lfps_decode_prefetch; the step shares its
    // call stamp, so an error raised ahead still fails this step
    if (!pp->pre_epoch)
      return fail(LFPS_E_INVALID, "LFPS_FLAG_PREFETCHED without a preceding lfps_decode_prefetch");
    c.epoch = pp->pre_epoch;
    c.prefetch = 1;
    pp->pre_epoch = 0;
    return enqueue_step(c, pp, sm, q, k_new, v_new, out_host, in_host, m_max);
  }
  pp->pre_epoch = 0;        // a full step changes the tables: an earlier prefetch is stale
  if (g_prof_on || !(c.flags & LFPS_FLAG_GRAPH)) {
    c.epoch = next_epoch();
    return enqueue_step(c, pp, sm, q, k_new, v_new, out_host, in_host, m_max);
  }
  // CUDA-graph step: replays a captured step when nothing baked into it has
  // changed (shapes, parameters, state and workspace, device buffers, the
  // select kernel's context bucket); the call stamp then comes from device
  // memory (ws.done[1], drawn by the step's first kernel)
  const int m_bucket = (m_max + 8191) / 8192 * 8192;
  GraphKey key;
  memset(&key, 0, sizeof(key));
  key.dims = *dims;
  key.params = *p;
  key.state = *st;
  key.ws = ws->base;
  key.q = q; key.k_new = k_new; key.v_new = v_new;
  key.m_bucket = m_bucket;
  key.has_in = in_host != nullptr;
  key.has_out = out_host != nullptr;
  c.epoch = 0;
  c.stamp = reinterpret_cast<const int*>(c.done + 1);
  if (!in_host) {
    // device inputs: copied into the pipe's staging buffer, so that one
    // graph serves callers whose input tensors change from step to step
    const size_t qb = (size_t)c.NS * c.d * 2, kb = (size_t)c.B * c.Hkv * c.d * 2;
    if (pp->stage_bytes < qb + 2 * kb) {
      if (pp->stage) {
        cudaStreamSynchronize(sm);
        cudaFree(pp->stage);
      }
      pp->stage = nullptr;
      pp->stage_bytes = 0;
      LAUNCH(cudaMalloc(&pp->stage, qb + 2 * kb));
      pp->stage_bytes = qb + 2 * kb;
    }
    char* st = static_cast<char*>(pp->stage);
    if (q != st) LAUNCH(cudaMemcpyAsync(st, q, qb, cudaMemcpyDeviceToDevice, sm));
    if (k_new != st + qb) LAUNCH(cudaMemcpyAsync(st + qb, k_new, kb, cudaMemcpyDeviceToDevice, sm));
    if (v_new != st + qb + kb)
      LAUNCH(cudaMemcpyAsync(st + qb + kb, v_new, kb, cudaMemcpyDeviceToDevice, sm));
    q = st;
    k_new = st + qb;
    v_new = st + qb + kb;
    key.q = q; key.k_new = k_new; key.v_new = v_new;
  }
  StepGraph* g = nullptr;
  for (size_t i = 0; i < pp->graphs.size(); ++i)
    if (pp->graphs[i]->key == key) {
      g = pp->graphs[i];
      pp->graphs.erase(pp->graphs.begin() + i);
      pp->graphs.push_back(g);
      break;
    }
  if (!g) {
    rc = capture_step(c, pp, key, q, k_new, v_new, out_host, in_host, m_bucket, &g);
    if (rc) return rc;
    if ((int)pp->graphs.size() == kMaxGraphs) {
      delete pp->graphs.front();
      pp->graphs.erase(pp->graphs.begin());
    }
    pp->graphs.push_back(g);
  }
  if (in_host && in_host != g->in_host) {
    LAUNCH(cudaGraphExecMemcpyNodeSetParams1D(g->exec, g->in_node, const_cast<void*>(q), in_host,
                                              g->in_bytes, cudaMemcpyHostToDevice));
    g->in_host = in_host;
  }
  if (out_host && out_host != g->out_host) {
    LAUNCH(cudaGraphExecMemcpyNodeSetParams1D(g->exec, g->out_node, out_host, c.out, g->out_bytes,
                                              cudaMemcpyDeviceToHost));
    g->out_host = out_host;
  }
  LAUNCH(cudaGraphLaunch(g->exec, sm));
  return LFPS_OK;
}

int lfps_exact_topk_step(const lfps_dims* dims, const lfps_params* p, const lfps_state* st,
                         const lfps_workspace* ws, const void* q, const int32_t* n_host,
                         void* stream) {
  lfps::Ctx c;
  int rc = make_ctx(dims, p, st, ws, &c);
  if (rc) return rc;
  if (!q) return fail(LFPS_E_INVALID, "q is NULL");
  int m_max = 0;
  rc = check_context(c, n_host, false, &m_max);
  if (rc) return rc;
  cudaStream_t sm = static_cast<cudaStream_t>(stream);
  const __nv_bfloat16* qb = static_cast<const __nv_bfloat16*>(q);
  LAUNCH_P("clear_err", sm, lfps::launch_clear_err(c, sm));
  LAUNCH_P("exact_score", sm, lfps::launch_exact_score(c, qb, m_max, sm));
  LAUNCH_P("exact_topk", sm, lfps::launch_topk(c, c.S, sm));
  LAUNCH_P("exact_attend", sm, lfps::launch_attend(c, qb, 1, sm));
  return LFPS_OK;
}

// ---- per-head stage API (k_stages.cu) -------------------------------------
#define STREAM(s) static_cast<cudaStream_t>(s)

int lfps_stage_logits(const double* keys, int32_t d, const int64_t* rows, int32_t nrows,
                      const double* q, double* out, void* stream) {
  if (!keys || !q || !out || d < 1 || nrows < 0) return fail(LFPS_E_INVALID, "stage_logits: bad arguments");
  if (nrows == 0) return LFPS_OK;
  LAUNCH(lfps::stage_logits(keys, d, rows, nrows, q, out, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_thresholds(const double* ver, const double* sla, int32_t m, double scale, double a,
                          int32_t materialize, double* out, double* scratch, void* stream) {
  if (!ver || !sla || !out || !scratch) return fail(LFPS_E_INVALID, "stage_thresholds: NULL argument");
  if (m < 2) return fail(LFPS_E_INVALID, "thresholds require at least 2 table slots");
  if (m > 512 * lfps::kBlk)   // tables.cuh kLeaves segments
    return fail(LFPS_E_UNSUPPORTED, "stage_thresholds: m <= %d", 512 * lfps::kBlk);
  LAUNCH(lfps::stage_thresholds(ver, sla, m, scale, a, materialize, out, scratch, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_candidates(int32_t mode, const double* ver, const double* sla, int32_t m,
                          double scale, const double* thr, const int64_t* in_idx, int32_t n_in,
                          const int32_t* offsets, int32_t n_off, int64_t base_index, int32_t n,
                          int32_t sink, int32_t window, int64_t* out_idx, int32_t* out_count,
                          void* stream) {
  if (mode < 0 || mode > 2 || !out_idx || !out_count) return fail(LFPS_E_INVALID, "stage_candidates: bad arguments");
  if (mode != 2 && (!ver || !sla || !thr || m < 0)) return fail(LFPS_E_INVALID, "stage_candidates: tables");
  if (mode != 0 && n_in > 0 && !in_idx) return fail(LFPS_E_INVALID, "stage_candidates: in_idx");
  if (mode == 1 && (!offsets || n_off < 1)) return fail(LFPS_E_INVALID, "stage_candidates: offsets");
  const long long U = mode == 2 ? n : m;
  if (U < 0 || (U + 31) / 32 * 4 > 200 * 1024) return fail(LFPS_E_UNSUPPORTED, "stage_candidates: universe too large");
  LAUNCH(lfps::stage_candidates(mode, ver, sla, m, scale, thr, in_idx, n_in, offsets, n_off, base_index,
                                n, sink, window, out_idx, out_count, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_topk(const int64_t* idx, const double* scores, int32_t p, int32_t k, int64_t* out_idx,
                    int32_t* out_count, void* stream) {
  if (!idx || !scores || !out_idx || !out_count || p < 1 || k < 1) return fail(LFPS_E_INVALID, "stage_topk: bad arguments");
  LAUNCH(lfps::stage_topk(idx, scores, p, k, out_idx, out_count, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_attend(const double* keys, const double* values, int32_t d, const int64_t* idx,
                      int32_t nidx, const double* q, double* out, double* weights, int32_t* err,
                      void* stream) {
  if (!keys || !values || !q || !out || !weights || !err || d < 1 || nidx < 1)
    return fail(LFPS_E_INVALID, "stage_attend: bad arguments");
  LAUNCH(lfps::stage_attend(keys, values, d, idx, nidx, q, out, weights, err, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_update(double* ver, double* sla, int32_t base, int32_t m, const int64_t* sel,
                      const double* weights, int32_t k, int32_t renorm, double rf, double scale,
                      int64_t* clamps, double* tmp, void* stream) {
  if (!ver || !sla || !sel || !weights || !clamps || !tmp || k < 1 || base < 1 || m < 0)
    return fail(LFPS_E_INVALID, "stage_update: bad arguments");
  LAUNCH(lfps::stage_update(ver, sla, base, m, sel, weights, k, renorm, rf, scale,
                            reinterpret_cast<long long*>(clamps), tmp, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_grow(double* ver, double* sla, int32_t base, int32_t m, int32_t carry, void* stream) {
  if (!ver || !sla || m < 0 || base < 0) return fail(LFPS_E_INVALID, "stage_grow: bad arguments");
  LAUNCH(lfps::stage_grow(ver, sla, base, m, carry, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_init_tables(const double* w, int32_t s, int32_t m, double r, double* ver, double* sla,
                           void* stream) {
  if (!w || !ver || !sla || s < 1 || m < 1) return fail(LFPS_E_INVALID, "stage_init_tables: bad arguments");
  LAUNCH(lfps::stage_init_tables(w, s, m, r, ver, sla, STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_head_stats(const double* keys, const double* values, int32_t n, int32_t d, int32_t sink,
                          const double* q, double* mean_key, double* mean_value, double* sigma,
                          double* tmp, int32_t* err, void* stream) {
  if (!keys || !values || !q || !mean_key || !mean_value || !sigma || !tmp || !err || d < 1)
    return fail(LFPS_E_INVALID, "stage_head_stats: bad arguments");
  if (n <= sink + 1) return fail(LFPS_E_INVALID, "need more than sink_count + 1 = %d rows, have %d", sink + 1, n);
  LAUNCH(lfps::stage_head_stats(keys, values, n, d, sink, q, mean_key, mean_value, sigma, tmp, err,
                                STREAM(stream)));
  return LFPS_OK;
}

int lfps_stage_gate(const double* keys, const double* values, int32_t n, int32_t d, int32_t sink,
                    int32_t window, const double* q, const double* mean_key, const double* mean_value,
                    double sigma, int32_t bypass_mode, double* out, int32_t* err, void* stream) {
  if (!keys || !values || !q || !mean_key || !mean_value || !out || !err || d < 1)
    return fail(LFPS_E_INVALID, "stage_gate: bad arguments");
  if (sink < 1 || sink > 31 || window < 1 || window > 64)
    return fail(LFPS_E_UNSUPPORTED, "stage_gate: sink_count in [1, 31], local_window in [1, 64]");
  if (n <= sink + window) return fail(LFPS_E_INVALID, "context shorter than sink_count + local_window");
  LAUNCH(lfps::stage_gate(keys, values, n, d, sink, window, q, mean_key, mean_value, sigma, bypass_mode,
                          out, err, STREAM(stream)));
  return LFPS_OK;
}

int lfps_overlap(const lfps_dims* dims, const int32_t* sel, const int32_t* sel_cnt,
                 const int32_t* exact, const int32_t* exact_cnt, int32_t list_stride,
                 int32_t cnt_stride, double* eta, void* stream) {
  int rc = check_dims(dims);
  if (rc) return rc;
  if (!sel || !sel_cnt || !exact || !exact_cnt || !eta) return fail(LFPS_E_INVALID, "NULL argument");
  if (list_stride < 1 || cnt_stride < 1) return fail(LFPS_E_INVALID, "bad strides");
  lfps::Ctx c;
  memset(&c, 0, sizeof(c));
  c.B = dims->batch; c.Hkv = dims->kv_heads; c.G = dims->group;
  c.Hq = c.Hkv * c.G; c.NS = c.B * c.Hq;
  LAUNCH(lfps::launch_overlap(c, sel, sel_cnt, exact, exact_cnt, list_stride, cnt_stride, eta,
                              static_cast<cudaStream_t>(stream)));
  return LFPS_OK;
}

}  // extern "C"

int lfps_check_dims(const lfps_dims* d) { return check_dims(d); }
