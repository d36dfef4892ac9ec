"""Paged K/V caches for a serving caller (lfps_kv_pool_*).

The decode kernels address ``lfps_state.k_cache / v_cache`` as contiguous
bf16 ``[B, Hkv, n_max, d]``.  ``KvPool`` reserves that range as virtual
address space and maps physical pages (the device's allocation granularity,
2 MiB) per (request, KV head) only as its context grows -- the GPU's MMU is
the page table, so the hot path is unchanged -- and unmaps a finished
request's pages.  The reference keeps one KvStore per head whose arrays
double and copy when full (``store.py:8-90``, ``_grow`` at :79-90); here a
context grows by mapping one more page, with no copy and no re-pointing of
the kernels, for a batch of long-context requests on one 180 GB device.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib

SLACK_ROWS = 64            # rows past the context backed for a kernel's last row tile


class _CudaArray:
    """__cuda_array_interface__ view of a raw device range (int16 payload)."""

    def __init__(self, ptr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": shape, "typestr": "<i2",
                                         "data": (ptr, False), "version": 2, "strides": None}


def page_bytes() -> int:
    lib = _lib.load_library()
    n = int(lib.lfps_kv_pool_page_bytes())
    if n <= 0:
        _lib.check(n, "lfps_kv_pool_page_bytes")
    return n


def page_rows(d: int) -> int:
    """Rows of one (request, KV head) per physical page at head dim d."""
    return page_bytes() // (2 * d)


class KvPool:
    """Virtual [B, Hkv, n_max, d] K and V caches backed page by page.

    n_max * d * 2 must be a multiple of the page size (``page_rows(d)`` rows;
    BatchedSession(paged=True) rounds n_max up).  ``k`` / ``v`` are bf16
    tensor views of the whole virtual range: only rows a ``reserve`` covered
    may be touched."""

    def __init__(self, dims: _lib.Dims, device: torch.device):
        self.lib = _lib.load_library()
        self.dims = dims
        self.device = device
        self._h = C.c_void_p()
        kp, vp = C.c_void_p(), C.c_void_p()
        with torch.cuda.device(device):
            _lib.check(self.lib.lfps_kv_pool_create(C.byref(dims), C.byref(self._h),
                                                     C.byref(kp), C.byref(vp)), "kv pool")
        shape = (dims.batch, dims.kv_heads, dims.n_max, dims.d)
        self.k = torch.as_tensor(_CudaArray(kp.value, shape), device=device).view(torch.bfloat16)
        self.v = torch.as_tensor(_CudaArray(vp.value, shape), device=device).view(torch.bfloat16)
        self.rows_per_page = page_bytes() // (2 * dims.d)
        self.backed = [0] * dims.batch          # rows usable per request (all heads)

    def _on_device(self):
        """The pool's device current for a C call (the caller may be on another)."""
        import contextlib
        dev = getattr(self, "device", None)
        return torch.cuda.device(dev) if dev is not None else contextlib.nullcontext()

    def reserve(self, b: int, rows: int) -> None:
        """Back rows [0, rows) (+ the kernels' slack) of request b, all heads."""
        if rows <= self.backed[b]:
            return
        with self._on_device():
            for h in range(self.dims.kv_heads):
                _lib.check(self.lib.lfps_kv_pool_reserve(self._h, b, h, rows), "kv pool reserve")
        want = min(rows + SLACK_ROWS, self.dims.n_max)
        pages = -(-want // self.rows_per_page)
        self.backed[b] = (self.dims.n_max if want >= self.dims.n_max
                          else pages * self.rows_per_page - SLACK_ROWS)

    def release(self, b: int) -> None:
        """Unmap request b's pages (its rows become inaccessible)."""
        with self._on_device():
            _lib.check(self.lib.lfps_kv_pool_release(self._h, b), "kv pool release")
        self.backed[b] = 0

    def mapped_bytes(self) -> int:
        return int(self.lib.lfps_kv_pool_mapped_bytes(self._h))

    def close(self) -> None:
        if self._h:
            self.k = self.v = None
            _lib.check(self.lib.lfps_kv_pool_destroy(self._h), "kv pool destroy")
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
