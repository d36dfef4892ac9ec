"""Host cost of the pieces of BatchedSession.decode_step_host at C1 (scratch
tool): each piece timed alone over many calls, then the whole call."""
import ctypes as C
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def per_call(fn, n=2000):
    fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    import torch
    from paper_2506_15704_b200.config import LfpsConfig
    from paper_2506_15704_b200.session import BatchedSession
    from paper_2506_15704_b200.workload import GqaSpec, populate
    dev = torch.device("cuda", 0)
    spec = GqaSpec(batch=1, kv_heads=8, group=4, d=128, n_prefill=16384, steps=32, seed=42)
    sess = BatchedSession(LfpsConfig(d=128), 1, 8, 4, n_max=16384 + 4096, device=dev)
    st = populate(sess, spec)
    sess.graph = True
    packed = torch.cat([st.q.reshape(32, -1), st.k_new.reshape(32, -1), st.v_new.reshape(32, -1)],
                       dim=1).cpu().pin_memory()
    inp = packed[0].clone().pin_memory()
    out = torch.empty(tuple(sess.out.shape), dtype=torch.float32).pin_memory()
    print("is_pinned          %.2f us" % per_call(lambda: inp.is_pinned()))
    print("current_stream     %.2f us" % per_call(lambda: sess._stream()))
    print("ctypes n_host      %.2f us" % per_call(lambda: (C.c_int32 * sess.B)(*sess.n_host)))
    print("_params            %.2f us" % per_call(lambda: sess._params(0.05, True, False)))
    print("result()           %.2f us" % per_call(lambda: sess.result()))
    print("data_ptr x2        %.2f us" % per_call(lambda: (inp.data_ptr(), out.data_ptr())))
    # whole steps, same input buffer (no memcpy-node update) and rotating buffers
    for name, src in (("same buffer", lambda t: inp), ("rotating", lambda t: packed[t % 32])):
        enq = []
        for t in range(400):
            x = src(t)
            t0 = time.perf_counter()
            sess.decode_step_host(x, 0.05, out_host=out)
            t1 = time.perf_counter()
            sess.wait_output()
            if t >= 20:
                enq.append((t1 - t0) * 1e6)
        enq.sort()
        print("decode_step_host (%s): median enqueue %.1f us" % (name, enq[len(enq) // 2]))
    lib = sess.lib
    print("ctypes abi_version %.2f us" % per_call(lambda: lib.lfps_abi_version()))
    # the C-ABI step call alone (prepared arguments; same buffers every call)
    from paper_2506_15704_b200 import _lib
    n_host = (C.c_int32 * sess.B)(*sess.n_host)
    args = (C.byref(sess.dims), C.byref(sess._params(0.05, True, False)), C.byref(sess.state),
            C.byref(sess.ws), C.c_void_p(inp.data_ptr()), C.c_void_p(sess._in_dev.data_ptr()
            if sess._in_dev is not None else 0), n_host, C.c_void_p(out.data_ptr()), sess._stream())
    if sess._in_dev is not None:
        ts = []
        for t in range(300):
            n_host[0] = sess.n_host[0]
            t0 = time.perf_counter()
            _lib.check(lib.lfps_decode_step_host_io(*args), "step")
            t1 = time.perf_counter()
            lib.lfps_wait_output(C.byref(sess.ws))
            sess.n_host = [n + 1 for n in sess.n_host]
            if t >= 20:
                ts.append((t1 - t0) * 1e6)
        ts.sort()
        print("C-ABI step call alone: median %.1f us" % ts[len(ts) // 2])
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
