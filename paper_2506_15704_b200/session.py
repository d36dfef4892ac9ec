"""BatchedSession: device-resident LFPS state for B requests x Hq query heads.

This is the B200 form of the reference's per-head ``HeadSession``
(engine.py:38-47): one object owns, for one attention layer,

* the bf16 KV cache [B, Hkv, n_max, d] shared by each KV head's G query
  heads (GQA; the reference's sessions each own a private fp64 KvStore),
* every (request, q-head) session's fp64 tracker tables (vertical table and
  slash ring), lazy scale, ring base and clamp counter,
* the frozen gate priors (K-bar, V-bar per KV head, sigma^2 per q-head),
* one workspace of per-step scratch and results.

All arithmetic runs in liblfps_b200.so (csrc/); this module only allocates
device memory with torch and passes raw pointers across the C-ABI.  Torch is
plumbing here, not the product: no torch op touches the decode path.
"""

from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .config import LfpsConfig

_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)
from .errors import DeviceError, LfpsError

CNT_C0, CNT_C1, CNT_PROBE, CNT_DROP, CNT_K, CNT_C2, CNT_CLAMP, CNT_BLOCKS = range(8)


def make_params(cfg: LfpsConfig, k_fraction: float, export_sets: bool = False,
                trace: bool = False, split: bool = False, graph: bool = False,
                prefetched: bool = False) -> _lib.Params:
    err = cfg.device_limits_error()
    if err:
        raise ValueError(err)
    p = _lib.Params()
    p.r, p.epsilon, p.a = cfg.r, cfg.epsilon, cfg.a
    p.k_fraction = float(k_fraction)
    p.sqrt_d = math.sqrt(cfg.d)
    p.sqrt_d_f32 = float(torch.tensor(math.sqrt(cfg.d), dtype=torch.float32))
    p.s, p.sink_count, p.local_window = cfg.s, cfg.sink_count, cfg.local_window
    p.bypass_mode = 1 if cfg.bypass_mode == "mean_only" else 0
    p.exhaustive = 1 if cfg.exhaustive_fallback else 0
    offs = sorted(set(cfg.expansion_offsets))
    p.n_offsets = len(offs)
    for i, o in enumerate(offs):
        p.offsets[i] = o
    p.flags = ((_lib.FLAG_EXPORT_SETS if export_sets else 0) | (_lib.FLAG_TRACE if trace else 0)
               | (_lib.FLAG_SPLIT if split else 0) | (_lib.FLAG_GRAPH if graph else 0)
               | (_lib.FLAG_PREFETCHED if prefetched else 0))
    return p


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


@dataclass
class BatchedStepResult:
    """Device views of one step's results (valid until the next step)."""

    output: torch.Tensor       # f32 [B, Hq, d]
    rho: torch.Tensor          # f64 [B, Hq]
    bypassed: torch.Tensor     # i32 [B, Hq]
    counts: torch.Tensor       # i32 [B, Hq, 8]: c0 c1 probe c0_dropped k c2 clamps blocks
    c2_idx: torch.Tensor       # i32 [B, Hq, list_cap] (first counts[..., 5] valid)
    c2_score: torch.Tensor     # f32 [B, Hq, list_cap]
    err: torch.Tensor          # i32 [1 + B*Hq]


class BatchedSession:
    """Device state of one layer for B requests (see module docstring)."""

    def __init__(self, cfg: LfpsConfig, batch: int, kv_heads: int, group: int, n_max: int,
                 m_cap: int | None = None, device: torch.device | str | None = None,
                 export_sets: bool = False, kv_cache: tuple | None = None,
                 paged: bool = False, kv_blocks: tuple | None = None):
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        device = torch.device(device)
        if device.type != "cuda":
            raise DeviceError("BatchedSession needs a CUDA device (no CPU fallback)")
        if device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = device
        err = cfg.device_limits_error()
        if err:
            raise ValueError(err)
        self.lib = _lib.load_library()
        self.cfg = cfg
        self.export_sets = export_sets
        self.trace = False          # LFPS_FLAG_TRACE: per-session phase timestamps
        self.split = True           # LFPS_FLAG_SPLIT: two session halves on two streams
        # LFPS_FLAG_GRAPH: a step is one CUDA-graph launch.  It cuts the host's
        # enqueue time (C4 ~100 -> ~60 us) but the replayed step runs slower on
        # the device than the stream-launched kernels (PDL overlap, the input
        # staging copies); so by default only the host-input path, where the
        # host is on the critical path of every step, uses it
        self.graph = True           # decode_step_host
        self.graph_device = False   # decode_step
        self.B, self.Hkv, self.G = batch, kv_heads, group
        self.Hq = kv_heads * group
        self.NS = batch * self.Hq
        self.d = cfg.d
        self.n_max = int(n_max)
        self.block_table = None
        if kv_blocks is not None:
            # a serving caller's block-table cache: (k_pool, v_pool, block_table,
            # block_rows), pools bf16 [blocks, block_rows, Hkv, d], table int32
            # [B, max_blocks] on the device; n_max = max_blocks * block_rows
            if paged or kv_cache is not None:
                raise ValueError("kv_blocks excludes paged=True and kv_cache")
            k_pool, v_pool, table, block_rows = kv_blocks
            block_rows = int(block_rows)
            if tuple(table.shape[:1]) != (batch,) or table.dtype != torch.int32:
                raise ValueError(f"block_table must be int32 [{batch}, max_blocks]")
            for t in (k_pool, v_pool):
                if (t.dim() != 4 or tuple(t.shape[1:]) != (block_rows, kv_heads, cfg.d)
                        or t.dtype != torch.bfloat16):
                    raise ValueError(f"kv pools must be bf16 [blocks, {block_rows}, {kv_heads}, "
                                     f"{cfg.d}]")
            self.block_table = table.contiguous()
            self.block_rows = block_rows
            self.n_max = int(table.shape[1]) * block_rows
            n_max = self.n_max
        if paged:
            # whole pages per (request, KV head): round n_max up
            from .kv_pool import page_rows
            with torch.cuda.device(device):
                pr = page_rows(cfg.d)
            self.n_max = -(-self.n_max // pr) * pr
        m_cap = int(m_cap if m_cap is not None else n_max - cfg.sink_count + 2)
        m_cap += m_cap & 1
        self.m_cap = m_cap
        self.dims = _lib.Dims(batch, kv_heads, group, cfg.d, self.n_max, m_cap)
        self.layout = _lib.workspace_layout(self.dims)
        self.sla_cap = _lib.slash_capacity(self.dims)
        dev = self.device
        f64, i32 = torch.float64, torch.int32
        self.kv_pool = None
        if paged:
            if kv_cache is not None:
                raise ValueError("paged=True allocates its own KV pool")
            from .kv_pool import KvPool
            self.kv_pool = KvPool(self.dims, dev)
            self.k_cache, self.v_cache = self.kv_pool.k, self.kv_pool.v
        elif kv_blocks is not None:
            self.k_cache, self.v_cache = kv_blocks[0], kv_blocks[1]
            if self.k_cache.device != dev or self.v_cache.device != dev:
                raise ValueError(f"kv pools must be on {dev}")
        elif kv_cache is not None:
            # an existing cache (e.g. one layer's rows reused by other layers'
            # trackers): bf16 [batch, kv_heads, n_max, d] pair on this device
            self.k_cache, self.v_cache = kv_cache
            shape = (batch, kv_heads, self.n_max, cfg.d)
            for t in (self.k_cache, self.v_cache):
                if tuple(t.shape) != shape or t.dtype != torch.bfloat16 or t.device != dev:
                    raise ValueError(f"kv_cache tensors must be bf16 {shape} on {dev}")
        else:
            self.k_cache = torch.zeros(batch, kv_heads, self.n_max, cfg.d, dtype=torch.bfloat16,
                                       device=dev)
            self.v_cache = torch.zeros_like(self.k_cache)
        self.n_ctx = torch.zeros(batch, dtype=i32, device=dev)
        self.n_host = [0] * batch
        self.ver = torch.zeros(self.NS, m_cap, dtype=f64, device=dev)
        self.sla = torch.zeros(self.NS, self.sla_cap, dtype=f64, device=dev)
        self.scale = torch.ones(self.NS, dtype=f64, device=dev)
        self.sla_base = torch.zeros(self.NS, dtype=i32, device=dev)
        self.clamp_count = torch.zeros(self.NS, dtype=torch.int64, device=dev)
        self.mean_key = torch.zeros(batch * kv_heads, cfg.d, dtype=f64, device=dev)
        self.mean_value = torch.zeros_like(self.mean_key)
        self.sigma_hat_sq = torch.zeros(self.NS, dtype=f64, device=dev)
        self.ws_buf = torch.zeros(self.layout.total_bytes, dtype=torch.uint8, device=dev)
        self.state = _lib.State(_ptr(self.k_cache), _ptr(self.v_cache), _ptr(self.n_ctx),
                                _ptr(self.ver), _ptr(self.sla), _ptr(self.scale),
                                _ptr(self.sla_base), _ptr(self.clamp_count),
                                _ptr(self.mean_key), _ptr(self.mean_value),
                                _ptr(self.sigma_hat_sq),
                                _ptr(self.block_table) if self.block_table is not None else None,
                                self.block_rows if self.block_table is not None else 0,
                                int(self.block_table.shape[1]) if self.block_table is not None
                                else 0)
        self.ws = _lib.Workspace(_ptr(self.ws_buf), self.layout.total_bytes)
        self._views()
        self.step_count = 0
        self.tables_stale = False
        self._in_dev = None        # decode_step_host's device staging buffer
        self._in_dev_ptr = None
        self._pin_cache = {}       # decode_step_host: pinned-ness per base tensor (weak)
        self._out_checked = None   # decode_step_host: the last checked output buffer (weak)
        self._in_bytes = None
        self._released = set()     # paged: requests whose pages were returned

    # -- workspace views ----------------------------------------------------
    def _region(self, off: int, dtype, shape):
        nbytes = torch.empty((), dtype=dtype).element_size()
        count = 1
        for s in shape:
            count *= s
        return self.ws_buf[off: off + count * nbytes].view(dtype).view(*shape)

    def _views(self):
        L, NS, B, Hq = self.layout, self.NS, self.B, self.Hq
        cap = L.list_cap
        self.rho = self._region(L.rho, torch.float64, (B, Hq))
        self.bypass = self._region(L.bypass, torch.int32, (B, Hq))
        self.err = self._region(L.err, torch.int32, (NS + 1,))
        self.out = self._region(L.out, torch.float32, (B, Hq, self.d))
        self.thr = self._region(L.thr, torch.float64, (B, Hq, 2, 4))
        self.counts = self._region(L.counts, torch.int32, (B, Hq, 8))
        self.bits = self._region(L.bits, torch.int32, (NS, 2, L.words))
        self.probe_idx = self._region(L.probe_idx, torch.int32, (B, Hq, cap))
        self.probe_score = self._region(L.probe_score, torch.float32, (B, Hq, cap))
        self.c2_idx = self._region(L.c2_idx, torch.int32, (B, Hq, cap))
        self.c2_score = self._region(L.c2_score, torch.float32, (B, Hq, cap))
        self.trace_buf = self._region(L.trace, torch.int64, (NS, 16))

    def _stream(self):
        # the raw handle of torch's current stream (a tenth of the cost of
        # building a torch.cuda.Stream for it: this is on every step's path)
        if _RAW_STREAM is not None:
            idx = self.device.index
            return C.c_void_p(_RAW_STREAM(torch.cuda.current_device() if idx is None else idx))
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _params(self, k_fraction: float = 1.0, graph: bool = False,
                prefetched: bool = False) -> _lib.Params:
        # the C side only reads the struct: one per distinct argument set
        # (building it costs ~14 us of Python, a third of a C1 step); the
        # last set is checked first by identity (hashing the config is slower)
        flags = (self.export_sets, self.trace, self.split, graph, prefetched)
        last = self.__dict__.get("_params_last")
        if (last is not None and last[0] is self.cfg and last[1] == k_fraction
                and last[2] == flags):
            return last[3]
        key = (self.cfg, float(k_fraction)) + flags
        cache = self.__dict__.setdefault("_params_cache", {})
        p = cache.get(key)
        if p is None:
            if len(cache) > 64:
                cache.clear()
            p = cache[key] = make_params(self.cfg, k_fraction, self.export_sets, self.trace,
                                         self.split, graph, prefetched)
        self._params_last = (self.cfg, k_fraction, flags, p)
        return p

    # -- bootstrap ----------------------------------------------------------
    def load_prefill(self, b: int, keys: torch.Tensor, values: torch.Tensor):
        """Copy request b's prefill rows (bf16 [Hkv, n0, d]) into the cache."""
        n0 = keys.shape[1]
        if n0 >= self.n_max:
            raise ValueError("prefill longer than the KV cache")
        if n0 <= self.cfg.sink_count + self.cfg.s:
            raise ValueError(
                f"prefill needs more than sink_count + s = {self.cfg.sink_count + self.cfg.s} rows")
        self._back(b, n0 + 1, reload=True)
        for h in range(self.Hkv):
            self._kv_write(b, h, 0, keys[h], values[h])
        self.n_host[b] = n0
        self.n_ctx[b] = n0

    def load_unit(self, b: int, h: int, keys: torch.Tensor, values: torch.Tensor):
        """Copy one (request, KV-head) unit's prefill rows (bf16 [n0, d]);
        every unit of a request must be loaded with the same n0."""
        n0 = keys.shape[0]
        if n0 >= self.n_max:
            raise ValueError("prefill longer than the KV cache")
        if n0 <= self.cfg.sink_count + self.cfg.s:
            raise ValueError(
                f"prefill needs more than sink_count + s = {self.cfg.sink_count + self.cfg.s} rows")
        self._back(b, n0 + 1, reload=True)
        self._kv_write(b, h, 0, keys, values)
        self.n_host[b] = n0
        self.n_ctx[b] = n0

    def bootstrap_tables(self, s_begin: int, weights: torch.Tensor):
        """Eq. 4 seeding for sessions [s_begin, s_begin + count); weights
        f32 [count, s, m0] on the device (init_tables, tables.py:247-281)."""
        weights = weights.to(self.device, torch.float32).contiguous()
        count, s, m0 = weights.shape
        if s != self.cfg.s:
            raise ValueError(f"expected {self.cfg.s} prefill weight vectors, got {s}")
        _lib.check(self.lib.lfps_bootstrap_tables(
            C.byref(self.dims), C.byref(self._params()), C.byref(self.state), C.byref(self.ws),
            C.c_void_p(weights.data_ptr()), s_begin, count, m0, self._stream()),
            "bootstrap_tables")

    def bootstrap_stats(self, last_query: torch.Tensor, requests: tuple | None = None):
        """Freeze the gate priors (compute_head_stats, gate.py:51-74);
        last_query bf16 [B, Hq, d].  ``requests`` = (first, count) limits it
        to those requests (one reloaded into a running batch)."""
        lq = last_query.to(self.device, torch.bfloat16).contiguous()
        if requests is None:
            _lib.check(self.lib.lfps_bootstrap_stats(
                C.byref(self.dims), C.byref(self._params()), C.byref(self.state),
                C.byref(self.ws), C.c_void_p(lq.data_ptr()), self._stream()), "bootstrap_stats")
            return
        _lib.check(self.lib.lfps_bootstrap_stats_requests(
            C.byref(self.dims), C.byref(self._params()), C.byref(self.state), C.byref(self.ws),
            C.c_void_p(lq.data_ptr()), int(requests[0]), int(requests[1]), self._stream()),
            "bootstrap_stats")

    def clear_errors(self):
        self.err.zero_()

    def close(self):
        """Release the library's per-workspace streams and events
        (lfps_workspace_release); the session is unusable afterwards."""
        if getattr(self, "ws", None) is not None and self.lib is not None:
            with torch.cuda.device(self.device):
                _lib.check(self.lib.lfps_workspace_release(C.byref(self.ws)), "close")
            self.ws = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass

    def sync_host_counts(self):
        """Re-read the context lengths from the device (the committing kernel
        advances n_ctx; a failed step leaves it): the host mirror n_host is
        advanced optimistically by every enqueued step."""
        dev = [int(x) for x in self.n_ctx.cpu()]
        if dev != self.n_host:
            self.step_count -= 1
        self.n_host = dev

    def check_errors(self, what: str = "step"):
        """Raise the reference's exception for the first failed session.

        A failed step commits nothing (engine.py:8-9), so the host mirror of
        the context lengths is rolled back to the device's; a session-local
        failure of the commit (err[0] = -stamp) still appended the rows."""
        err = self.err.cpu()
        if int(err[0]) == 0:
            return
        self.sync_host_counts()
        # err[0] = the failed call's stamp (negated: a session-local failure),
        # err[1 + s] = stamp << 4 | code (codes of other calls are stale)
        stamp = abs(int(err[0]))
        raw = err[1:]
        live = (raw >> 4) == stamp
        codes = torch.where(live, raw & 15, torch.zeros_like(raw))
        bad = torch.nonzero(codes).flatten()
        s = int(bad[0]) if bad.numel() else -1
        code = int(codes[s]) if s >= 0 else 0
        msg = _lib.ERR_NAMES.get(code, f"device error {code}")
        if code == 3:
            raise ZeroDivisionError(f"{what}: session {s}: {msg}")
        raise ValueError(f"{what}: session {s}: {msg}")

    # -- decode ---------------------------------------------------------------
    def prefetch(self):
        """Run the q-independent half of the next decode step ahead
        (lfps_decode_prefetch): thresholds, C0, C1 and the probe sets of every
        session depend on the tables and the context only (engine.py:146-160),
        so they can be built on the current stream while the caller still
        computes the step's queries -- e.g. beside earlier layers of the
        model.  The next decode_step / decode_step_host must pass
        ``prefetched=True`` (same stream, or ordered after it)."""
        if self.tables_stale:
            raise ValueError("tables out of sync with the KV store (append_rows was used)")
        self._back_step()
        n_host = (C.c_int32 * self.B)(*self.n_host)
        _lib.check(self.lib.lfps_decode_prefetch(
            C.byref(self.dims), C.byref(self._params(1.0)), C.byref(self.state), C.byref(self.ws),
            n_host, self._stream()), "decode_prefetch")

    def decode_step(self, q: torch.Tensor, k_new: torch.Tensor, v_new: torch.Tensor,
                    k_fraction: float, check: bool = False,
                    out_host: torch.Tensor | None = None,
                    prefetched: bool = False) -> BatchedStepResult:
        """One LFPS decode step for all sessions (engine.py:97-201).

        q bf16 [B, Hq, d]; k_new, v_new bf16 [B, Hkv, d] (device).  On a
        data error no state is committed; ``check=True`` synchronises and
        raises it.  ``out_host`` (f32 [B, Hq, d], pinned host memory) receives
        the step's output as soon as it is final, copied beside the commit
        kernel (lfps_decode_step_host_out); it is filled once the current
        stream passes this call.  ``prefetched``: the candidate sets were built
        by ``prefetch()`` (the step runs the gate, the finish and the commit)."""
        if not 0.0 < k_fraction <= 1.0:
            raise ValueError(f"k_fraction must be in (0, 1], got {k_fraction}")
        if self.tables_stale:
            raise ValueError("tables out of sync with the KV store (append_rows was used)")
        for name, t, shape in (("q", q, (self.B, self.Hq, self.d)),
                               ("new_key", k_new, (self.B, self.Hkv, self.d)),
                               ("new_value", v_new, (self.B, self.Hkv, self.d))):
            if tuple(t.shape) != shape:
                raise ValueError(f"{name} must have shape {shape}, got {tuple(t.shape)}")
            if t.dtype != torch.bfloat16 or t.device != self.device or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous bf16 tensor on {self.device}")
        self._back_step()
        n_host = (C.c_int32 * self.B)(*self.n_host)
        graph = self.graph_device and (out_host is None or out_host.is_pinned())
        params = self._params(k_fraction, graph and not prefetched, prefetched)
        if out_host is None:
            _lib.check(self.lib.lfps_decode_step(
                C.byref(self.dims), C.byref(params), C.byref(self.state),
                C.byref(self.ws), C.c_void_p(q.data_ptr()), C.c_void_p(k_new.data_ptr()),
                C.c_void_p(v_new.data_ptr()), n_host, self._stream()), "decode_step")
        else:
            if (tuple(out_host.shape) != tuple(self.out.shape) or out_host.dtype != torch.float32
                    or out_host.device.type != "cpu" or not out_host.is_contiguous()):
                raise ValueError(f"out_host must be a contiguous f32 CPU tensor of shape "
                                 f"{tuple(self.out.shape)}")
            _lib.check(self.lib.lfps_decode_step_host_out(
                C.byref(self.dims), C.byref(params), C.byref(self.state),
                C.byref(self.ws), C.c_void_p(q.data_ptr()), C.c_void_p(k_new.data_ptr()),
                C.c_void_p(v_new.data_ptr()), n_host, C.c_void_p(out_host.data_ptr()),
                self._stream()), "decode_step")
        self.n_host = [n + 1 for n in self.n_host]
        self.step_count += 1
        if check:
            torch.cuda.current_stream(self.device).synchronize()
            self.check_errors("decode_step")
        return self.result()

    def _kv_write(self, b: int, h: int, r0: int, keys: torch.Tensor, values: torch.Tensor):
        """Rows [r0, r0 + len) of unit (b, h) into the cache (plumbing)."""
        n = keys.shape[0]
        if self.block_table is None:
            self.k_cache[b, h, r0:r0 + n].copy_(keys)
            self.v_cache[b, h, r0:r0 + n].copy_(values)
            return
        r = torch.arange(r0, r0 + n, device=self.device)
        blk = self.block_table[b].long()[r // self.block_rows]
        off = r % self.block_rows
        self.k_cache[blk, off, h] = keys.to(self.device, torch.bfloat16)
        self.v_cache[blk, off, h] = values.to(self.device, torch.bfloat16)

    def kv_rows(self, b: int, h: int, n: int):
        """(K, V) bf16 [n, d] copies of unit (b, h)'s first n rows."""
        if self.block_table is None:
            return self.k_cache[b, h, :n].clone(), self.v_cache[b, h, :n].clone()
        r = torch.arange(n, device=self.device)
        blk = self.block_table[b].long()[r // self.block_rows]
        off = r % self.block_rows
        return self.k_cache[blk, off, h], self.v_cache[blk, off, h]

    # -- paged KV (kv_pool.py) ------------------------------------------------
    def _back(self, b: int, rows: int, reload: bool = False):
        """Paged caches: back rows [0, rows) of request b before they are
        written or read (the append of a step writes row n)."""
        if self.kv_pool is None:
            return
        if b in self._released and not reload:
            raise ValueError(f"request {b} was released; load_prefill it again first")
        self._released.discard(b)
        self.kv_pool.reserve(b, rows)

    def _back_step(self):
        if self.kv_pool is not None:
            for b in range(self.B):
                self._back(b, min(self.n_host[b] + 1, self.n_max))

    def release_request(self, b: int):
        """Paged caches: return request b's KV pages (a finished request).
        Its rows are gone; decoding the batch again needs a new prefill for b
        (load_prefill / load_unit + bootstrap)."""
        if self.kv_pool is None:
            raise ValueError("release_request needs paged=True")
        self.kv_pool.release(b)
        self._released.add(b)

    def kv_mapped_bytes(self) -> int:
        """Bytes of device memory behind the K and V caches."""
        if self.kv_pool is not None:
            return self.kv_pool.mapped_bytes()
        return 2 * self.k_cache.numel() * self.k_cache.element_size()

    def step_input_bytes(self) -> int:
        """Bytes of one step's packed host input (lfps_step_input_bytes)."""
        n = int(self.lib.lfps_step_input_bytes(C.byref(self.dims)))
        if n < 0:
            raise ValueError("invalid dims")
        return n

    def pack_step_inputs(self, q: torch.Tensor, k_new: torch.Tensor,
                         v_new: torch.Tensor) -> torch.Tensor:
        """Pinned host bf16 buffer [q | k_new | v_new] for decode_step_host."""
        parts = [t.detach().to("cpu", torch.bfloat16).reshape(-1) for t in (q, k_new, v_new)]
        packed = torch.cat(parts).pin_memory()
        if packed.numel() * 2 != self.step_input_bytes():
            raise ValueError("q / k_new / v_new do not have the session's shapes")
        return packed

    def decode_step_host(self, inputs_host: torch.Tensor, k_fraction: float,
                         out_host: torch.Tensor | None = None,
                         check: bool = False, prefetched: bool = False) -> BatchedStepResult:
        """decode_step with host inputs (lfps_decode_step_host_io):
        ``inputs_host`` is a contiguous CPU bf16 tensor packed as
        [q | k_new | v_new] (``pack_step_inputs``; pinned for an asynchronous
        copy).  The library copies it into the session's device staging
        buffer on an internal stream that overlaps the step's table
        statistics; ``out_host`` as in decode_step."""
        if not 0.0 < k_fraction <= 1.0:
            raise ValueError(f"k_fraction must be in (0, 1], got {k_fraction}")
        if self.tables_stale:
            raise ValueError("tables out of sync with the KV store (append_rows was used)")
        # (the checks cost more than the C-ABI call: the pinned-ness of the
        # buffers' base tensors and the output buffer's checks are cached
        # per tensor object -- a decode loop passes views of one pinned
        # input buffer and the same output buffer every step)
        nbytes = self._in_bytes
        if nbytes is None:
            nbytes = self._in_bytes = self.step_input_bytes()
        if (not inputs_host.is_cpu or inputs_host.dtype is not torch.bfloat16
                or inputs_host.numel() * 2 != nbytes or not inputs_host.is_contiguous()):
            raise ValueError(f"inputs_host must be a contiguous bf16 CPU tensor of "
                             f"{nbytes // 2} elements")
        pinned = self._pinned(inputs_host)
        out_ptr = None
        if out_host is not None:
            ent = self._out_checked
            if (ent is None or ent[0]() is not out_host or ent[1] != out_host.data_ptr()
                    or out_host.numel() != ent[3]):
                if (tuple(out_host.shape) != tuple(self.out.shape)
                        or out_host.dtype != torch.float32 or not out_host.is_cpu
                        or not out_host.is_contiguous()):
                    raise ValueError(f"out_host must be a contiguous f32 CPU tensor of shape "
                                     f"{tuple(self.out.shape)}")
                ent = self._out_checked = (weakref.ref(out_host), out_host.data_ptr(),
                                           C.c_void_p(out_host.data_ptr()), out_host.numel())
            out_ptr = ent[2]
            pinned = pinned and self._pinned(out_host)
        self._back_step()
        if self._in_dev is None:
            self._in_dev = torch.empty(nbytes // 2, dtype=torch.bfloat16, device=self.device)
            self._in_dev_ptr = C.c_void_p(self._in_dev.data_ptr())
        n_host = (C.c_int32 * self.B)(*self.n_host)
        graph = self.graph and pinned
        _lib.check(self.lib.lfps_decode_step_host_io(
            C.byref(self.dims), C.byref(self._params(k_fraction, graph and not prefetched, prefetched)),
            C.byref(self.state), C.byref(self.ws), C.c_void_p(inputs_host.data_ptr()),
            self._in_dev_ptr, n_host, out_ptr, self._stream()), "decode_step")
        self.n_host = [n + 1 for n in self.n_host]
        self.step_count += 1
        if check:
            torch.cuda.current_stream(self.device).synchronize()
            self.check_errors("decode_step")
        return self.result()

    def _pinned(self, t: torch.Tensor) -> bool:
        """t.is_pinned(), cached per base tensor (views share their base's
        storage)."""
        base = t._base if t._base is not None else t
        ent = self._pin_cache.get(id(base))
        if ent is not None and ent[0]() is base:
            return ent[1]
        p = base.is_pinned()
        if len(self._pin_cache) >= 16:
            self._pin_cache.clear()
        self._pin_cache[id(base)] = (weakref.ref(base), p)
        return p

    def wait_output(self):
        """Block until the last host-output step's output (``out_host`` of
        decode_step_host / decode_step) is in host memory
        (lfps_wait_output).  Its commit may still be running on the device:
        an autoregressive loop needs only the output before it builds the next
        step's queries, and the next step is stream-ordered after the commit."""
        _lib.check(self.lib.lfps_wait_output(C.byref(self.ws)), "wait_output")

    def copy_tracker_from(self, other: "BatchedSession"):
        """Take over another session's tracker state, priors and context
        counts (same dims): e.g. one layer's bootstrap reused by other layers.
        The block summaries of this session's workspace are rebuilt by its
        first step."""
        if (self.B, self.Hkv, self.G, self.m_cap, self.sla_cap) != \
                (other.B, other.Hkv, other.G, other.m_cap, other.sla_cap):
            raise ValueError("sessions differ in shape")
        if self.kv_pool is not None:
            raise ValueError("copy_tracker_from shares another session's KV rows: not with "
                             "paged=True (pass kv_cache instead)")
        for name in ("ver", "sla", "scale", "sla_base", "clamp_count", "mean_key", "mean_value",
                     "sigma_hat_sq", "n_ctx"):
            getattr(self, name).copy_(getattr(other, name))
        self.n_host = list(other.n_host)
        self.ws_buf.zero_()

    def append_rows(self, k_new: torch.Tensor, v_new: torch.Tensor):
        """Append one K/V row per unit WITHOUT an LFPS step (store.append,
        store.py:64-77): the replay of the exact and full-attention reference
        modes (replay.run_trace).  The tracker tables no longer match the
        context afterwards, so further LFPS steps on this session raise."""
        for name, t in (("new_key", k_new), ("new_value", v_new)):
            if tuple(t.shape) != (self.B, self.Hkv, self.d) or t.dtype != torch.bfloat16:
                raise ValueError(f"{name} must be bf16 [{self.B}, {self.Hkv}, {self.d}]")
        self._back_step()
        for b in range(self.B):
            n = self.n_host[b]
            if n >= self.n_max:
                raise ValueError(f"request {b}: KV cache full")
            for h in range(self.Hkv):
                self._kv_write(b, h, n, k_new[b, h][None], v_new[b, h][None])
        self.n_ctx += 1
        self.n_host = [n + 1 for n in self.n_host]
        self.tables_stale = True

    def rollback_host_count(self):
        """Undo the host mirror advance after a step that committed nothing
        (kept for callers of round 1; check_errors now does this itself)."""
        self.sync_host_counts()

    def gate_near_epsilon(self, tol: float = 1e-12) -> torch.Tensor:
        """Sessions of the last step whose sink share rho lies within `tol`
        of epsilon (bool [B, Hq]).  The gate's fp64 exp is the canonical
        devmath.cexp, not libm's, so a rho this close to epsilon is where the
        bypass decision could differ from the reference's;
        such decisions are reported, not hidden."""
        return (self.rho - self.cfg.epsilon).abs() <= tol

    def result(self) -> BatchedStepResult:
        return BatchedStepResult(output=self.out, rho=self.rho, bypassed=self.bypass,
                                 counts=self.counts, c2_idx=self.c2_idx,
                                 c2_score=self.c2_score, err=self.err)

    def exact_topk_step(self, q: torch.Tensor, k_fraction: float) -> BatchedStepResult:
        """Exact full-scan Top-k over the current rows (bench.py:73-80);
        read-only on the tracker state.  Results reuse the workspace."""
        if not 0.0 < k_fraction <= 1.0:
            raise ValueError(f"k_fraction must be in (0, 1], got {k_fraction}")
        if tuple(q.shape) != (self.B, self.Hq, self.d) or q.dtype != torch.bfloat16:
            raise ValueError("q must be bf16 [B, Hq, d]")
        n_host = (C.c_int32 * self.B)(*self.n_host)
        _lib.check(self.lib.lfps_exact_topk_step(
            C.byref(self.dims), C.byref(self._params(k_fraction)), C.byref(self.state),
            C.byref(self.ws), C.c_void_p(q.contiguous().data_ptr()), n_host, self._stream()),
            "exact_topk_step")
        return self.result()

    def full_attention(self, q: torch.Tensor) -> torch.Tensor:
        """Exact softmax attention over every cached row of every session
        (full_attention_oracle, attention.py:88-97) on the device: the exact
        path with k_fraction = 1 selects all non-sink rows and attends them
        jointly with the sinks.  Returns a copy of the f32 [B, Hq, d] output;
        the workspace lists and counts are overwritten (like exact_topk_step)."""
        return self.exact_topk_step(q, 1.0).output.clone()

    def overlap(self, sel_idx: torch.Tensor, sel_counts: torch.Tensor,
                exact_idx: torch.Tensor, exact_counts: torch.Tensor) -> torch.Tensor:
        """eta per session (overlap_ratio, attention.py:116-124) for two
        [B, Hq, cap] index lists with [B, Hq, 8]-strided counts (slot 5)."""
        eta = torch.empty(self.B, self.Hq, dtype=torch.float64, device=self.device)
        cap = sel_idx.shape[-1]
        if exact_idx.shape[-1] != cap:
            raise ValueError("lists must share a capacity")
        _lib.check(self.lib.lfps_overlap(
            C.byref(self.dims), C.c_void_p(sel_idx.data_ptr()),
            C.c_void_p(sel_counts.data_ptr() + 4 * CNT_C2), C.c_void_p(exact_idx.data_ptr()),
            C.c_void_p(exact_counts.data_ptr() + 4 * CNT_C2), cap, sel_counts.shape[-1],
            C.c_void_p(eta.data_ptr()), self._stream()), "overlap")
        return eta

    # -- host snapshots (tests, diagnostics) ---------------------------------
    def session_tables(self, s: int):
        """(ver phys [m], sla phys [m] in logical order, scale) of session s."""
        b = s // self.Hq
        m = self.n_host[b] - self.cfg.sink_count
        base = int(self.sla_base[s])
        return (self.ver[s, :m].cpu().numpy(), self.sla[s, base: base + m].cpu().numpy(),
                float(self.scale[s]))

    def c2_list(self, b: int, qh: int):
        k = int(self.counts[b, qh, CNT_C2])
        return self.c2_idx[b, qh, :k].cpu().numpy()

    def _bitmap_list(self, b: int, qh: int, which: int):
        if not self.export_sets:
            raise LfpsError("C0/C1 sets are exported only with export_sets=True")
        m = self.n_host[b] - 1 - self.cfg.sink_count     # the step just taken
        words = self.bits[b * self.Hq + qh, which, : (m + 31) // 32].cpu().numpy()
        bits = np.unpackbits(words.view(np.uint8), bitorder="little")[:m]
        return np.nonzero(bits)[0].astype(np.int64) + self.cfg.sink_count

    def c0_list(self, b: int, qh: int):
        """C0 of the last step (absolute indices), export_sets sessions only."""
        return self._bitmap_list(b, qh, 0)

    def c1_list(self, b: int, qh: int):
        """C1 of the last step (absolute indices), export_sets sessions only."""
        return self._bitmap_list(b, qh, 1)

    def probe_list(self, b: int, qh: int):
        p = int(self.counts[b, qh, CNT_PROBE])
        return self.probe_idx[b, qh, :p].cpu().numpy()
