"""A/B of the CUDA-graph decode step (scratch tool): per-step host wall time
(synchronous) and device time of back-to-back steps, graph on / off, for
fixed device input buffers and for packed pinned host inputs."""
import sys
import time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_15704_b200.config import LfpsConfig
from paper_2506_15704_b200.session import BatchedSession
from paper_2506_15704_b200.workload import GqaSpec, populate

cfgname = sys.argv[1] if len(sys.argv) > 1 else "c1"
B, n0 = (1, 16384) if cfgname == "c1" else (64, 131072)
spec = GqaSpec(batch=B, kv_heads=8, group=4, d=128, n_prefill=n0, steps=16, seed=42)
sess = BatchedSession(LfpsConfig(d=128), B, 8, 4, n_max=n0 + 400, device="cuda")
st = populate(sess, spec)
qd, kd, vd = st.q[0].clone(), st.k_new[0].clone(), st.v_new[0].clone()
packed = [sess.pack_step_inputs(st.q[t], st.k_new[t], st.v_new[t]) for t in range(16)]
outh = torch.empty(sess.out.shape, dtype=torch.float32).pin_memory()
cs = torch.cuda.current_stream()
for graph in (False, True, False, True):
    sess.graph = graph
    # device inputs, fixed buffers, back to back
    for t in range(3):
        sess.decode_step(qd, kd, vd, 0.05)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    for t in range(30):
        qd.copy_(st.q[t % 16]); kd.copy_(st.k_new[t % 16]); vd.copy_(st.v_new[t % 16])
        sess.decode_step(qd, kd, vd, 0.05)
    e1.record()
    host_enq = (time.perf_counter() - h0) / 30 * 1e6
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / 30 * 1e3
    # host io, synchronous per step
    lat = []
    for t in range(30):
        a = time.perf_counter()
        sess.decode_step_host(packed[t % 16], 0.05, out_host=outh)
        cs.synchronize()
        lat.append(time.perf_counter() - a)
    lat.sort()
    sess.check_errors("ab")
    print(f"{cfgname} graph={graph}: device b2b {dev:.1f} us/step (host enqueue {host_enq:.1f} us), "
          f"host-io sync median {lat[15] * 1e6:.1f} us", flush=True)
