"""The C-ABI library loads on a CPU-only host and exports exactly what
include/lfps_b200.h declares; host-side validation rejects bad arguments
before anything touches a device (no compute calls here)."""

import ctypes as C
import os
import re

import pytest

from paper_2506_15704_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "lfps_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"LFPS_API\s+[\w\s\*]+?\b(lfps_\w+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for want in ("lfps_abi_version", "lfps_last_error", "lfps_workspace_layout",
                 "lfps_bootstrap_tables", "lfps_bootstrap_stats", "lfps_decode_step",
                 "lfps_decode_step_host_out", "lfps_decode_step_host_io",
                 "lfps_step_input_bytes", "lfps_exact_topk_step", "lfps_overlap",
                 "lfps_profile_enable",
                 "lfps_profile_collect", "lfps_decode_launches", "lfps_exact_launches",
                 "lfps_slash_capacity"):
        assert want in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) <= set(declared_functions())
    assert lib.lfps_abi_version() == _lib.ABI_VERSION
    assert lib.lfps_decode_launches(None, 0) == 5 and lib.lfps_exact_launches() > 0
    big = _lib.Dims(64, 8, 4, 128, 4096, 4096)
    assert lib.lfps_decode_launches(C.byref(big), _lib.FLAG_SPLIT) == 17   # 4 groups x 4 + commit
    assert lib.lfps_step_input_bytes(C.byref(big)) == (64 * 8 * 4 + 2 * 64 * 8) * 128 * 2
    assert lib.lfps_step_input_bytes(C.byref(_lib.Dims(0, 8, 4, 128, 4096, 4096))) < 0


def test_struct_layouts_match_header(tmp_path):
    """ctypes mirrors of the POD structs have the C compiler's sizes."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no C compiler")
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "lfps_b200.h"\nint main(void){printf("%zu %zu %zu '
                   '%zu %zu %zu", sizeof(lfps_dims), sizeof(lfps_params), sizeof(lfps_state), '
                   'sizeof(lfps_ws_layout), sizeof(lfps_workspace), sizeof(lfps_kernel_time));}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    c_sizes = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()]
    py_sizes = [C.sizeof(t) for t in (_lib.Dims, _lib.Params, _lib.State, _lib.WsLayout,
                                       _lib.Workspace, _lib.KernelTime)]
    assert c_sizes == py_sizes


def test_workspace_layout_regions_are_disjoint_and_aligned():
    dims = _lib.Dims(4, 8, 4, 128, 33000, 33000)
    lay = _lib.workspace_layout(dims)
    offs = sorted((getattr(lay, f), f) for f, _ in _lib.WsLayout._fields_
                  if f not in ("total_bytes", "words", "list_cap", "nblk", "dirty_words",
                               "scratch"))
    for (a, _), (b, _) in zip(offs, offs[1:]):
        assert b > a
    assert all(o % 256 == 0 for o, _ in offs)
    assert lay.total_bytes > offs[-1][0]
    assert lay.list_cap >= 33000 and lay.list_cap % 32 == 0 and lay.words * 32 >= 33000
    assert lay.nblk * 512 == _lib.slash_capacity(dims) >= 2 * 33000
    assert lay.dirty_words * 32 >= lay.nblk and lay.dirty_words <= 32


@pytest.mark.parametrize("bad", [
    dict(batch=0), dict(group=3), dict(d=100), dict(m_cap=33001), dict(n_max=1),
    dict(m_cap=510 * 512 + 2),
])
def test_invalid_dims_rejected_on_host(bad):
    kw = dict(batch=1, kv_heads=1, group=4, d=128, n_max=4096, m_cap=4096)
    kw.update(bad)
    with pytest.raises((ValueError, _lib.DeviceError)):
        _lib.workspace_layout(_lib.Dims(**kw))
    assert _lib.load_library().lfps_last_error()


def test_decode_step_validation_happens_before_launch():
    lib = _lib.load_library()
    dims = _lib.Dims(1, 1, 1, 64, 4096, 4096)
    p = _lib.Params()
    p.r, p.epsilon, p.a, p.k_fraction = 0.95, 0.85, 0.2, 1.5      # k_fraction out of range
    rc = lib.lfps_decode_step(C.byref(dims), C.byref(p), C.byref(_lib.State()),
                              C.byref(_lib.Workspace()), None, None, None, None, None)
    assert rc == -1
    assert b"k_fraction" in lib.lfps_last_error() or b"NULL" in lib.lfps_last_error() \
        or b"must" in lib.lfps_last_error()


def test_host_io_validation_happens_before_launch():
    lib = _lib.load_library()
    dims = _lib.Dims(1, 1, 1, 64, 4096, 4096)
    p = _lib.Params()
    buf = (C.c_uint8 * 64)()
    rc = lib.lfps_decode_step_host_io(C.byref(dims), C.byref(p), C.byref(_lib.State()),
                                      C.byref(_lib.Workspace()), None, C.byref(buf), None,
                                      None, None)
    assert rc == -1 and b"in_host" in lib.lfps_last_error()
    bad = _lib.Dims(1, 1, 1, 60, 4096, 4096)                      # d not a multiple of 16
    rc = lib.lfps_decode_step_host_io(C.byref(bad), C.byref(p), C.byref(_lib.State()),
                                      C.byref(_lib.Workspace()), C.byref(buf), C.byref(buf),
                                      None, None, None)
    assert rc < 0 and lib.lfps_step_input_bytes(C.byref(bad)) < 0


def test_kv_pool_validation_on_host():
    import torch
    lib = _lib.load_library()
    pool, kp, vp = C.c_void_p(), C.c_void_p(), C.c_void_p()
    bad = _lib.Dims(0, 1, 1, 64, 4096, 4096)
    assert lib.lfps_kv_pool_create(C.byref(bad), C.byref(pool), C.byref(kp), C.byref(vp)) < 0
    assert lib.lfps_kv_pool_reserve(None, 0, 0, 1) == -1
    assert lib.lfps_kv_pool_release(None, 0) == -1
    assert lib.lfps_kv_pool_destroy(None) == 0
    if not torch.cuda.is_available():       # no driver: the VM API is reported missing
        assert lib.lfps_kv_pool_page_bytes() < 0


def test_library_refuses_to_pretend_without_gpu():
    """No CPU fallback: constructing a device session off-GPU raises."""
    import torch
    from paper_2506_15704_b200 import DeviceError, LfpsConfig
    from paper_2506_15704_b200.session import BatchedSession
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises((DeviceError, RuntimeError, AssertionError)):
        BatchedSession(LfpsConfig(d=64), 1, 1, 1, n_max=1024, device="cuda")


def test_kv_pool_backed_rows_bookkeeping():
    """KvPool.reserve's host bookkeeping (no device): the rows usable without
    another map call follow the C side's page rounding with the 64-row
    slack, the last page of a span backs up to n_max, and release resets."""
    from paper_2506_15704_b200 import kv_pool

    calls = []

    class FakeLib:
        def lfps_kv_pool_reserve(self, h, b, kv, rows):
            calls.append((b, kv, rows))
            return 0

        def lfps_kv_pool_release(self, h, b):
            return 0

    pool = kv_pool.KvPool.__new__(kv_pool.KvPool)
    pool.lib, pool._h = FakeLib(), C.c_void_p(1)
    pool.dims = _lib.Dims(2, 2, 4, 128, 3 * 8192, 3 * 8192)
    pool.rows_per_page = 8192
    pool.backed = [0, 0]
    pool.reserve(0, 100)
    assert pool.backed[0] == 8192 - kv_pool.SLACK_ROWS and len(calls) == 2   # one call per head
    pool.reserve(0, 8128)                       # still inside the first page's usable rows
    assert len(calls) == 2
    pool.reserve(0, 8129)                       # crosses: two pages
    assert pool.backed[0] == 2 * 8192 - kv_pool.SLACK_ROWS and len(calls) == 4
    pool.reserve(0, 3 * 8192 - 10)              # the span's last page: everything backed
    assert pool.backed[0] == 3 * 8192
    pool.release(0)
    assert pool.backed[0] == 0 and pool.backed[1] == 0
    pool._h = C.c_void_p()                      # nothing to destroy
