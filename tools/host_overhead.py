"""Host-side cost of one end-to-end decode step at C1 (batch 1 x 16k): the
wall time of BatchedSession.decode_step_host (Python + C-ABI enqueue) and of
the wait for the output, against the whole step, over N steps.

    python tools/host_overhead.py [--steps 200] [--no-graph]
"""
import argparse
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--context", type=int, default=16384)
    ap.add_argument("--profile", action="store_true", help="cProfile the step loop")
    args = ap.parse_args()
    import torch
    from paper_2506_15704_b200.config import LfpsConfig
    from paper_2506_15704_b200.session import BatchedSession
    from paper_2506_15704_b200.workload import GqaSpec, populate
    dev = torch.device("cuda", 0)
    spec = GqaSpec(batch=args.batch, kv_heads=8, group=4, d=128, n_prefill=args.context,
                   steps=32, seed=42)
    sess = BatchedSession(LfpsConfig(d=128), args.batch, 8, 4,
                          n_max=args.context + args.steps + 64, device=dev)
    st = populate(sess, spec)
    sess.graph = not args.no_graph
    packed = torch.cat([st.q.reshape(32, -1), st.k_new.reshape(32, -1), st.v_new.reshape(32, -1)],
                       dim=1).cpu().pin_memory()
    out = torch.empty(tuple(sess.out.shape), dtype=torch.float32).pin_memory()
    enq, wait, tot = [], [], []
    prof = None
    if args.profile:
        import cProfile
        prof = cProfile.Profile()
        prof.enable()
    for t in range(args.steps):
        t0 = time.perf_counter()
        sess.decode_step_host(packed[t % 32], 0.05, out_host=out)
        t1 = time.perf_counter()
        sess.wait_output()
        t2 = time.perf_counter()
        if t >= 10:
            enq.append((t1 - t0) * 1e6)
            wait.append((t2 - t1) * 1e6)
            tot.append((t2 - t0) * 1e6)
    if prof:
        prof.disable()
        import pstats
        pstats.Stats(prof).sort_stats("tottime").print_stats(14)
    torch.cuda.synchronize()
    sess.check_errors("host overhead steps")
    med = statistics.median
    print(f"graph={not args.no_graph} batch={args.batch} ctx={args.context}: "
          f"enqueue {med(enq):.1f} us, wait {med(wait):.1f} us, step {med(tot):.1f} us (medians)")


if __name__ == "__main__":
    main()
