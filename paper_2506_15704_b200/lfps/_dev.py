"""Device plumbing of the per-head API: the current CUDA device and stream,
host <-> device copies, and the checked call into liblfps_b200.so.  Torch
only allocates and copies here; every stage's arithmetic is a kernel of
csrc/k_stages.cu (there is no CPU fallback)."""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from .. import _lib
from ..errors import DeviceError

F64 = torch.float64
I64 = torch.int64


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise DeviceError("the lfps device API needs a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def stream() -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr() if t is not None else None)


def f64(x, dev=None) -> torch.Tensor:
    """fp64 device copy of a host array (or a device tensor, cast)."""
    if isinstance(x, torch.Tensor):
        return x.to(dev or device(), F64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).to(dev or device())


def i64(x, dev=None) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(dev or device(), I64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x, dtype=np.int64)).to(dev or device())


def host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def call(name: str, *args) -> None:
    lib = _lib.load_library()
    _lib.check(getattr(lib, name)(*args), name)


ERR = {1: "non-finite logits in sparsity estimate", 2: "non-finite sparsity ratio",
       6: "zero-norm prefill query", 7: "softmax input contains non-finite scores"}


def raise_code(code: int) -> None:
    if code == 3:
        raise ZeroDivisionError("float division by zero")
    if code:
        raise ValueError(ERR.get(code, f"device error {code}"))
