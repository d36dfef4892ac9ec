#!/usr/bin/env python
"""LFPS decode-step benchmark on B200 (BASELINE.json metric).

Metric: LFPS index + sparse-attention microseconds per decode step per
layer (lower is better), with the HBM roofline of the dominant kernel, Top-k
recall eta against the exact full-scan path, and the reference's CPU path
timed on this host beside it.

Workload (default, ``--config c4``): BASELINE.json config 4 -- batch 64 x
128k context, Llama-3.1-8B attention shapes (32 query / 8 KV heads, d=128),
one layer, Top-k 5%, synthetic planted vertical/slash structure (torch
restatement of the reference generator, paper_2506_15704_b200/workload.py).
Under torchrun the 64 requests are sharded over the ranks (no collective on
the decode path); the step time is the max over ranks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the reference algorithm's CPU implementation on the
host cores (the oracle port of pkg/src/lfps, numpy, BLAS pinned to one thread
per worker process, one process per core) on the same config.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (batch, context, kv_heads, group, d, frac, description)
    "c4": (64, 131072, 8, 4, 128, 0.05,
           "C4: batch 64 x 128k context, Llama-3.1-8B shapes (32 q / 8 kv heads, d=128), "
           "1 layer, Top-k 5%"),
    "c2": (4, 32768, 8, 4, 128, 0.05,
           "C2: batch 4 x 32k context, Llama-3.1-8B shapes, 1 layer, Top-k 5%"),
    "c3": (16, 131072, 8, 4, 128, 0.05,
           "C3: batch 16 x 128k context, all 32 layers, Llama-3.1-8B shapes, Top-k 5%"),
    "c1": (1, 16384, 8, 4, 128, 0.05,
           "C1: batch 1 x 16k context, Llama-3.1-8B shapes, 1 layer, Top-k 5%"),
    # one rank's share of C4 on 2 / 4 / 8 GPUs (request split), on one GPU
    "c4s2": (32, 131072, 8, 4, 128, 0.05, "C4 per-rank share at 2 GPUs: batch 32 x 128k, 1 layer, Top-k 5%"),
    "c4s4": (16, 131072, 8, 4, 128, 0.05, "C4 per-rank share at 4 GPUs: batch 16 x 128k, 1 layer, Top-k 5%"),
    "c4s8": (8, 131072, 8, 4, 128, 0.05, "C4 per-rank share at 8 GPUs: batch 8 x 128k, 1 layer, Top-k 5%"),
}
METRIC = "LFPS index+sparse-attn us/decode-step/layer"
UNIT = "us/step"


def parse():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="c4")
    ap.add_argument("--recall-steps", type=int, default=3)
    ap.add_argument("--cpu-steps", type=int, default=6, help="steps per CPU worker sample")
    ap.add_argument("--cpu-workers", type=int, default=0, help="0 = all host cores")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--prefetch", action="store_true",
                    help="C3: each layer's candidate sets built ahead on a second stream "
                         "(lfps_decode_prefetch), the layers' gate/finish/commit in order")
    ap.add_argument("--no-graph", action="store_true",
                    help="e2e: enqueue each host-input step kernel by kernel (no CUDA graph)")
    ap.add_argument("--no-split", action="store_true",
                    help="disable LFPS_FLAG_SPLIT (two session halves on two streams)")
    ap.add_argument("--paged", action="store_true",
                    help="K/V in a KvPool (2 MiB pages mapped as contexts grow; kv_pool.py)")
    ap.add_argument("--no-gather", action="store_true",
                    help="N > 1: skip the final all-gather of outputs and C2 counts in e2e")
    ap.add_argument("--verify", type=int, default=2,
                    help="after the run, replay this many (request, KV-head) units of rank 0 "
                         "through the CPU oracle and require bit-exact tables and sets")
    ap.add_argument("--profile-only", action="store_true",
                    help="short run for ncu: no e2e, recall or cpu legs")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing
# ---------------------------------------------------------------------------

def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def dist_init(world, local):
    """One process per GPU over NCCL.  LFPS_DIST_BACKEND=gloo (with ranks
    sharing devices round-robin) exercises the multi-rank path on a box with
    fewer GPUs than ranks; timings from such a run are not scaling numbers."""
    import torch
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("LFPS_DIST_BACKEND", "nccl")
        dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)


def dist_backend() -> str:
    import torch.distributed as dist
    return dist.get_backend() if dist.is_initialized() else "none"


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _reduce(world, x: float, op: str) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def allmax(world, x: float) -> float:
    """Max over ranks (the step time of a multi-GPU run)."""
    return _reduce(world, x, "max")


def allsum(world, x: float) -> float:
    return _reduce(world, x, "sum")


def shard_requests(batch: int, world: int, rank: int) -> tuple[int, int]:
    """(requests on this rank, first request index): the batch is split into
    contiguous request ranges; every (request, KV-head) unit is independent,
    so no collective is needed on the decode path."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, extra = divmod(batch, world)
    count = base + (1 if rank < extra else 0)
    first = rank * base + min(rank, extra)
    if count < 1:
        raise SystemExit(f"batch {batch} is smaller than the {world} ranks")
    return count, first


# ---------------------------------------------------------------------------
# clocks (sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"lfps_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
            return
        t0 = time.time()                   # the timed region starts once sampling runs
        while time.time() - t0 < 5.0:
            if os.path.exists(self.path) and os.path.getsize(self.path) > 0:
                break
            time.sleep(0.02)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# CPU leg: the UNMODIFIED reference package (pkg/src/lfps, installed into
# baseline/_ref by tools/install_reference.sh) on the host's physical cores,
# one process per core, BLAS pinned to one thread before numpy loads.
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_BLAS_VARS = ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS",
              "NUMEXPR_NUM_THREADS", "VECLIB_MAXIMUM_THREADS")


def reference_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "lfps", "engine.py"))


def _cpu_worker(job):
    """One host core: one (request, KV-head) unit of the workload as the
    reference runs it -- G independent HeadSessions over identical bf16-valued
    K/V (the reference has no GQA) -- stepping the stock
    lfps.decode_step (engine.py:97-201) and timing lfps.bench.exact_topk_step
    (bench.py:73-80) on the same pre-append rows.  Inputs are generated before
    any timing; nothing of this repo runs inside the timed calls."""
    for var in _BLAS_VARS:
        os.environ[var] = "1"
    import numpy as np
    import torch
    torch.set_num_threads(1)
    from paper_2506_15704_b200.workload import GqaSpec, gen_unit
    spec = GqaSpec(**job["spec"])
    b, h, steps, warm, frac = job["b"], job["h"], job["steps"], job["warmup"], job["frac"]
    G, n0 = job["sessions"], spec.n_prefill
    u = gen_unit(spec, b, h, device="cpu")
    keys = u.keys.double().numpy()
    values = u.values.double().numpy()
    weights = u.weights.double().numpy()
    finals = u.final_query.double().numpy()
    qs = u.queries.double().numpy()              # [G, steps, d]
    del u
    if job["kind"] == "reference":
        sys.path.insert(0, REF_DIR)
        import lfps
        from lfps.bench import exact_topk_step
        cfg = lfps.LfpsConfig(d=spec.d)
        sessions = [lfps.prefill_bootstrap(keys[:n0], values[:n0], weights[g], finals[g], cfg)
                    for g in range(G)]

        def lfps_step(g, q, t):
            lfps.decode_step(sessions[g], q, keys[n0 + t], values[n0 + t], frac, cfg)

        def exact_step(g, q):
            st = sessions[g].store
            exact_topk_step(q, st, max(1, round(frac * st.n)), cfg.sink_count)
    else:                                        # the oracle port (reference arithmetic)
        from oracle import lfps_oracle as lo
        from paper_2506_15704_b200.config import LfpsConfig
        cfg = LfpsConfig(d=spec.d)
        kv, trs, prs = lo.bootstrap_unit(keys[:n0], values[:n0], weights[:G], finals[:G], cfg,
                                         lo.RefArith)
        kvs = [kv] + [lo.UnitKV(kv.keys.copy(), kv.values.copy(), kv.n) for _ in range(G - 1)]

        def lfps_step(g, q, t):
            lo.session_step(kvs[g], trs[g], prs[g], q, frac, cfg, lo.RefArith, "fp64")
            kvs[g].append(keys[n0 + t], values[n0 + t])

        def exact_step(g, q):
            lo.exact_topk_step(kvs[g], q, lo.budget_k(frac, kvs[g].n), cfg, "fp64")
    lfps_ns, exact_ns = [], []
    for t in range(warm + steps):
        for g in range(G):
            q = qs[g, t]
            t0 = time.perf_counter_ns()
            exact_step(g, q)
            t1 = time.perf_counter_ns()
            lfps_step(g, q, t)
            t2 = time.perf_counter_ns()
            if t >= warm:
                exact_ns.append(t1 - t0)
                lfps_ns.append(t2 - t1)
    return {"lfps_ns": lfps_ns, "exact_ns": exact_ns}


def physical_cores() -> int:
    """Physical cores available to this process (lscpu cores x sockets,
    capped by the affinity mask)."""
    avail = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        f = {k.strip(): v.strip() for k, v in (ln.split(":", 1) for ln in out.splitlines()
                                              if ":" in ln)}
        phys = int(f["Core(s) per socket"]) * int(f["Socket(s)"])
        return max(1, min(phys, avail or phys))
    except Exception:  # noqa: BLE001
        return max(1, avail or 1)


def cpu_leg(cfg_name: str, steps: int, warmup: int, workers: int, sessions: int = 2):
    """Time the reference's CPU path on the host cores; returns a dict.

    Bounded sample: each worker process steps `sessions` reference sessions
    of one unit for `steps` timed steps (+ warm-up); the per-layer-step time
    is extrapolated from the median session-step over all of a layer's
    sessions spread over the cores."""
    import multiprocessing as mp
    batch, ctx, hkv, group, d, frac, _ = CONFIGS[cfg_name]
    for var in _BLAS_VARS:
        os.environ[var] = "1"
    cores = workers or physical_cores()
    kind = "reference" if reference_available() else "port"
    sessions = min(sessions, group)
    spec = dict(batch=batch, kv_heads=hkv, group=group, d=d, n_prefill=ctx,
                steps=warmup + steps, seed=42)
    jobs = [dict(spec=spec, b=(i // hkv) % batch, h=i % hkv, steps=steps, warmup=warmup,
                 frac=frac, sessions=sessions, kind=kind) for i in range(cores)]
    ctxm = mp.get_context("spawn")
    t0 = time.time()
    with ctxm.Pool(cores) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.time() - t0
    lfps = [x for r in res for x in r["lfps_ns"]]
    exact = [x for r in res for x in r["exact_ns"]]
    ns_total = batch * hkv * group
    med_l = statistics.median(lfps) / 1e3
    med_e = statistics.median(exact) / 1e3
    per_worker = math.ceil(ns_total / cores)
    what = ("the unmodified reference package (baseline/_ref/lfps: decode_step, "
            "bench.exact_topk_step)" if kind == "reference" else
            "the oracle port at reference arithmetic (baseline/_ref missing)")
    return {
        "kind": kind,
        "session_step_us_median": med_l,
        "exact_session_step_us_median": med_e,
        "layer_step_us": med_l * per_worker,
        "exact_layer_step_us": med_e * per_worker,
        "cores": cores,
        "sessions_timed": len(lfps),
        "wall_s": wall,
        "sample": (f"{what}: {cores} worker processes (one per physical core, BLAS 1 thread) x "
                   f"{sessions} sessions of one (request, KV-head) unit x {steps} timed steps "
                   f"(+{warmup} warm-up) at context {ctx}; per-layer-step time extrapolated as "
                   f"median session-step x ceil({ns_total} sessions / {cores} cores)"),
    }


def cpu_model():
    try:
        out = subprocess.run("lscpu | grep 'Model name'", shell=True, capture_output=True,
                             text=True).stdout
        return out.split(":", 1)[1].strip()
    except Exception:  # noqa: BLE001
        return "unknown"


def run_reference(args, world, rank):
    if rank != 0:
        return
    # each timed "step" of this arm is a bounded sample: at most 24 steps per
    # worker (the reference's KV store doubles its capacity 64 rows past the
    # prefill), so --steps K --warmup W finishes within minutes at 128k
    r = cpu_leg(args.config, min(args.steps, 24), min(args.warmup, 2), args.cpu_workers)
    batch, ctx, hkv, group, d, frac, desc = CONFIGS[args.config]
    line = {
        "impl": "reference",
        "metric": METRIC, "value": r["layer_step_us"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": r["layer_step_us"] / 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "batch": batch, "context": ctx, "q_heads": hkv * group,
                   "kv_heads": hkv, "d": d, "topk_fraction": frac},
        "cpu_baseline": {"value": r["layer_step_us"], "unit": UNIT, "cores": r["cores"],
                         "kind": r["kind"], "sample": r["sample"], "cpu": cpu_model()},
        "e2e": {"value": r["layer_step_us"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "exact_topk_us_per_layer_step": r["exact_layer_step_us"],
        "session_step_us_median": r["session_step_us_median"],
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def step_bytes(sess, cfg) -> dict:
    """Algorithmic HBM bytes of the last decode step, per kernel.

    Counted from the step's actual sets, each byte once, at the kernel that
    must move it:

    * stats  -- the table blocks it read (rebuilt dirty blocks + hot blocks,
      4 KiB each, CNT_BLOCKS), the window's block summaries (32 B moments +
      8 B max per 512-slot segment, both tables), its C0 word lists;
    * select -- the C0 words (8 B per word entry, bounded by |C0|), the mean
      filter F at the candidate slots (both tables, 16 B per C1 slot), the
      probe list (4 B);
    * finish -- DISTINCT K rows of the unit's probe sets and V rows of its
      C2 sets plus sinks (the G q-heads of a unit share one row store), q
      in and out, the C2 list and scores;
    * update -- C2 scores + indices, the table read-modify-write (2 tables x
      16 B), the unit's K/V append;
    * gate   -- sink and local K rows per unit, q, K-bar / V-bar.

    ``reference`` is SURVEY.md §8(d)'s byte count for the reference algorithm
    (both fp64 tables read in full every step), for comparison."""
    import torch
    from paper_2506_15704_b200.session import CNT_BLOCKS, CNT_C0, CNT_C1, CNT_C2, CNT_PROBE
    B, Hkv, G, d, S = sess.B, sess.Hkv, sess.G, sess.d, cfg.sink_count
    counts = sess.counts.to(torch.int64)
    probe, c2, blocks = counts[..., CNT_PROBE], counts[..., CNT_C2], counts[..., CNT_BLOCKS]
    c0, c1 = counts[..., CNT_C0], counts[..., CNT_C1]
    active = (sess.bypass == 0)
    n_max = max(sess.n_host)
    row = d * 2

    def distinct(idx, cnt):
        # rows touched per unit: union over the unit's G sessions, plus sinks
        U = B * Hkv
        cap = idx.shape[-1]
        pos = torch.arange(cap, device=idx.device)
        li = idx.reshape(U, G, cap).to(torch.int64)
        ok = pos[None, None, :] < cnt.reshape(U, G)[..., None]
        mark = torch.zeros(U, n_max + 1, dtype=torch.bool, device=idx.device)
        uid = torch.arange(U, device=idx.device)[:, None, None].expand_as(li)
        mark[uid[ok], li[ok]] = True
        mark[:, :S] = True
        return mark.sum(1).to(torch.float64)

    k_rows = distinct(sess.probe_idx, probe * active)
    v_rows = distinct(sess.c2_idx, c2 * active)
    nseg = torch.tensor([(n - 1 - S) / 512 + 1 for n in sess.n_host], dtype=torch.float64,
                        device=counts.device).repeat_interleave(Hkv * G).reshape(B, Hkv * G)
    stats = blocks.double() * 512 * 8 + 2 * nseg * 40 + c0.double() * 8
    select = (c0.double() * 8 + c1.double() * 16 + probe.double() * 4) * active
    fin = ((k_rows.sum() + v_rows.sum()) * row + sess.NS * (row + d * 4)
           + float((c2 * active).sum()) * 8)
    upd = float(((c2.double() * (8 + 2 * 16)) * active).sum()) + B * Hkv * 2 * row
    gate = B * Hkv * (S + cfg.local_window) * row + sess.NS * (row + 8 * d) + B * Hkv * 2 * 8 * d
    kern = {"gate": float(gate), "stats": float(stats.sum()), "select": float(select.sum()),
            "finish": float(fin), "update": float(upd)}
    total = sum(kern.values())
    m = torch.tensor([n - 1 - S for n in sess.n_host], dtype=torch.float64)
    ref = float((m * 16).sum()) * Hkv * G + float(((probe + c2) * active).sum()) * row
    return {"kernels": kern, "total": total, "reference": ref,
            "blocks_mean": float(blocks.double().mean()),
            "k_rows_unit": float(k_rows.mean()), "v_rows_unit": float(v_rows.mean())}


def phase_trace(sess, step, t, dev) -> dict:
    """One extra (untimed) step with LFPS_FLAG_TRACE: mean per-CTA phase
    durations of the select and finish kernels (clock64, us at the max SM
    clock) and each kernel's span over all CTAs (globaltimer)."""
    import torch
    sess.trace = True
    sess.trace_buf.zero_()
    step(t)
    torch.cuda.synchronize(dev)
    sess.trace = False
    tr = sess.trace_buf.cpu().double()[sess.bypass.flatten().cpu() == 0]
    ghz = 1.965

    def us(col):
        return float(col.mean()) / ghz / 1e3

    return {
        # stats kernel (per session x table; table 0's CTA): A, A + B, A + B +
        # C; select kernel (per session): C0 assembly, + D
        "select": {"A_rebuild": us(tr[:, 1]), "B_merge": us(tr[:, 2] - tr[:, 1]),
                   "C_hot": us(tr[:, 7] - tr[:, 2]), "C0_assemble": us(tr[:, 3]),
                   "D_probe": us(tr[:, 4] - tr[:, 3]), "D_first_F_reads": us(tr[:, 6] - tr[:, 3]),
                   "cta_total": us(tr[:, 7] + tr[:, 4]),
                   "span": float(tr[:, 12].max() - tr[:, 15].min()) / 1e3},
        "finish": {"union": us(tr[:, 11]), "rows": us(tr[:, 8]), "merge": us(tr[:, 9] - tr[:, 8]),
                   "checks": us(tr[:, 10] - tr[:, 9]), "cta_total": us(tr[:, 10]),
                   "span": float(tr[:, 14].max() - tr[:, 13].min()) / 1e3},
        "note": "mean per-CTA phase time (clock64 at 1.965 GHz) and kernel span (globaltimer) "
                "of one extra untimed step"}


def verify_units(sess, spec, stream, step_log, cfg, frac, count, dev) -> dict:
    """Replay `count` (request, KV-head) units of this run through the CPU
    oracle (oracle/lfps_oracle.py, canonical device arithmetic) from their
    bootstrap over every decode step the bench executed, and require the
    device's final tracker tables (phys values, lazy scale, clamp counts)
    to be bit-identical, the last step's probe and C2 sets and counts equal,
    its output within 1e-5 relative L2, and the KV rows the device appended
    equal to the step inputs.  Identical final tables imply identical C2
    sets on every step (every update folds its C2 set into both tables).
    Runs after all timing; the oracle is only the checker here."""
    import numpy as np
    import torch
    from oracle import lfps_oracle as lo
    from paper_2506_15704_b200.session import CNT_C2, CNT_PROBE
    from paper_2506_15704_b200.workload import gen_unit
    t0 = time.time()
    B, Hkv, G, S = sess.B, sess.Hkv, sess.G, cfg.sink_count
    n0 = spec.n_prefill
    units = []
    for i in range(count):
        b = (i * max(1, B - 1)) // max(1, count - 1) if count > 1 else 0
        units.append((min(b, B - 1), (3 * i + 1) % Hkv))
    worst = 0.0
    checked = []
    for b, h in dict.fromkeys(units):
        u = gen_unit(spec, b, h, device=dev)
        n_end = sess.n_host[b]
        assert n_end == n0 + len(step_log)
        keys = sess.k_cache[b, h, :n_end].double().cpu().numpy()
        vals = sess.v_cache[b, h, :n_end].double().cpu().numpy()
        np.testing.assert_array_equal(keys[:n0], u.keys[:n0].double().cpu().numpy())
        kv, trs, prs = lo.bootstrap_unit(keys[:n0], vals[:n0], u.weights.double().cpu().numpy(),
                                         u.final_query.double().cpu().numpy(), cfg, lo.DevArith)
        qs = stream.q[:, b, h * G:(h + 1) * G].double().cpu().numpy()      # [T_in, G, d]
        kn = stream.k_new[:, b, h].double().cpu().numpy()
        vn = stream.v_new[:, b, h].double().cpu().numpy()
        outs = None
        for j, t in enumerate(step_log):
            np.testing.assert_array_equal(keys[n0 + j], kn[t], err_msg=f"appended K row {j}")
            np.testing.assert_array_equal(vals[n0 + j], vn[t], err_msg=f"appended V row {j}")
            outs = lo.unit_step(kv, trs, prs, qs[t], kn[t], vn[t], frac, cfg, lo.DevArith, "fp32")
        out = sess.out[b, h * G:(h + 1) * G].double().cpu().numpy()
        cnt = sess.counts[b, h * G:(h + 1) * G].cpu().numpy()
        for g in range(G):
            s = b * sess.Hq + h * G + g
            ver, sla, sc = sess.session_tables(s)
            tag = f"unit ({b}, {h}) q-head {g}"
            assert sc == trs[g].scale, tag
            np.testing.assert_array_equal(ver, trs[g].ver_view(), err_msg=tag + " ver")
            np.testing.assert_array_equal(sla, trs[g].sla_view(), err_msg=tag + " sla")
            assert int(sess.clamp_count[s]) == trs[g].clamp_count, tag
            o = outs[g]
            if not o.bypassed:
                assert cnt[g, CNT_PROBE] == o.probe.size and cnt[g, CNT_C2] == o.c2.size, tag
                np.testing.assert_array_equal(sess.probe_list(b, h * G + g), o.probe, err_msg=tag)
                np.testing.assert_array_equal(sess.c2_list(b, h * G + g), o.c2, err_msg=tag)
            err = np.linalg.norm(out[g] - o.output) / max(np.linalg.norm(o.output), 1e-12)
            assert err <= 1e-5, (tag, err)
            worst = max(worst, err)
        checked.append([b, h])
    return {"units": checked, "sessions": len(checked) * G, "steps": len(step_log),
            "tables": "bit-exact (phys ver/sla, scale, clamp counts) after every step's update",
            "last_step_sets": "probe and C2 bit-exact", "output_rel_err_max": worst,
            "oracle": "oracle/lfps_oracle.py DevArith (pinned against the reference, tests/)",
            "seconds": time.time() - t0}


def run_ours(args, world, rank, local):
    import ctypes as C
    import numpy as np
    import torch
    from paper_2506_15704_b200 import _lib
    from paper_2506_15704_b200.config import LfpsConfig
    from paper_2506_15704_b200.session import CNT_BLOCKS, CNT_C2, CNT_PROBE, BatchedSession
    from paper_2506_15704_b200.sharded import ShardedSession, populate_sharded
    from paper_2506_15704_b200.workload import GqaSpec, StepStream

    batch, ctx, hkv, group, d, frac, desc = CONFIGS[args.config]
    e2e_steps = 0 if args.profile_only else args.steps
    recall_steps = 0 if args.profile_only else args.recall_steps
    prof_steps = min(args.steps, 8)
    gather_steps = args.steps if world > 1 and not args.profile_only else 0
    T = args.warmup + args.steps + gather_steps + prof_steps + 1 + e2e_steps + recall_steps
    T_in = min(T, 64)          # distinct synthetic step inputs, cycled
    cfg = LfpsConfig(d=d)
    # one spec for the whole batch: every unit is generated from its own seed,
    # so the union of the ranks' units is exactly the single-GPU workload
    spec = GqaSpec(batch=batch, kv_heads=hkv, group=group, d=d, n_prefill=ctx, steps=T_in,
                   seed=42)
    dev = torch.device("cuda", torch.cuda.current_device())
    t_setup = time.time()
    # (request, KV-head) units partitioned over the ranks (sharded.plan_shards:
    # requests when B >= P, KV heads when B < P); no collective on the path
    ss = ShardedSession(cfg, batch, hkv, group, n_max=ctx + T + 8, rank=rank, world=world,
                        device=dev, paged=args.paged)
    sess = ss.sess
    b_local = ss.shard.nb
    full = populate_sharded(ss, spec)
    stream = StepStream(q=torch.stack([ss.local_q(x) for x in full.q]),
                        k_new=torch.stack([ss.local_kv(x) for x in full.k_new]),
                        v_new=torch.stack([ss.local_kv(x) for x in full.v_new]))
    del full
    sess.split = not args.no_split
    sess.graph = not args.no_graph
    setup_s = time.time() - t_setup
    cuda_stream = torch.cuda.current_stream(dev)

    step_log = []              # input index of every decode step, in order (--verify)

    def step(t):
        t %= T_in
        step_log.append(t)
        sess.decode_step(stream.q[t], stream.k_new[t], stream.v_new[t], frac)

    for t in range(args.warmup):
        step(t)
    torch.cuda.synchronize(dev)
    sess.check_errors("warm-up")
    n_before = list(sess.n_host)

    # ---- timed region: device-resident inputs, no instrumentation ----
    # every step is bracketed by its own events; L2 is flushed (a 512 MiB
    # write, 4x the 126 MB L2) before each one, outside the brackets
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier(world)
    torch.cuda.synchronize(dev)
    for i, t in enumerate(range(args.warmup, args.warmup + args.steps)):
        flush.fill_(i & 255)
        evs[i][0].record(cuda_stream)
        step(t)
        evs[i][1].record(cuda_stream)
    torch.cuda.synchronize(dev)
    barrier(world)
    clock_info = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms_local = sum(step_ms) / args.steps
    del flush
    sess.check_errors("timed steps")
    ms = allmax(world, ms_local)

    # ---- N > 1: the same steps, each followed by the final all-gather of the
    # batch's outputs and C2 counts (ShardedSession.gather), device-timed ----
    gather_ms = None
    if gather_steps:
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        barrier(world)
        torch.cuda.synchronize(dev)
        g0.record(cuda_stream)
        for t in range(args.warmup + args.steps, args.warmup + args.steps + gather_steps):
            step(t)
            ss.gather(with_c2=False)
        g1.record(cuda_stream)
        torch.cuda.synchronize(dev)
        barrier(world)
        gather_ms = allmax(world, g0.elapsed_time(g1) / gather_steps)

    # ---- per-kernel CUDA events on the launch stream (separate pass) ----
    prof_base = args.warmup + args.steps + gather_steps
    _lib.profile_enable(True)
    for t in range(prof_base, prof_base + prof_steps):
        step(t)
    torch.cuda.synchronize(dev)
    _lib.profile_enable(False)
    kt = _lib.profile_collect()
    sess.check_errors("profiled steps")
    phases = phase_trace(sess, step, prof_base + prof_steps - 1, dev)

    # ---- algorithmic bytes per kernel (last profiled step) and the roofline ----
    peak, peak_src = measured_peaks()
    alg = step_bytes(sess, cfg)
    kernel_ms = {k: v[1] / max(1, v[0]) for k, v in kt.items()}
    dominant = max(kernel_ms, key=kernel_ms.get)
    dom_ms = kernel_ms[dominant]
    dom_bytes = alg["kernels"].get(dominant, 0)
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic_all = {}
    tpath = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
    if os.path.exists(tpath) and args.config == "c4":
        with open(tpath) as f:
            traffic_all = {k: v.get("traffic_bytes") for k, v in json.load(f)["kernels"].items()}
    traffic = traffic_all.get(dominant)
    per_kernel = {}
    for k, ms_k in kernel_ms.items():
        by = alg["kernels"].get(k, 0.0)
        gbs = by / (ms_k * 1e-3) / 1e9
        per_kernel[k] = {"ms": ms_k, "algorithmic_bytes": by, "GBps": gbs, "frac": gbs / peak,
                         "ncu_traffic_bytes": traffic_all.get(k)}
    counts = sess.counts.cpu().numpy()
    bypass = int(sess.bypass.sum())
    probe = counts[..., CNT_PROBE].astype(np.int64)
    c2 = counts[..., CNT_C2].astype(np.int64)

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if e2e_steps:
        # each step's q | k_new | v_new packed in one pinned host buffer
        # (BatchedSession.pack_step_inputs' layout): one H2D copy per step
        nq, nk = stream.q[0].numel(), stream.k_new[0].numel()
        packed = torch.cat([stream.q.reshape(T_in, -1), stream.k_new.reshape(T_in, -1),
                            stream.v_new.reshape(T_in, -1)], dim=1)
        inh = packed.cpu().pin_memory()
        ind = torch.empty_like(packed[0])
        qd = ind[:nq].view(stream.q[0].shape)
        kd = ind[nq:nq + nk].view(stream.k_new[0].shape)
        vd = ind[nq + nk:].view(stream.v_new[0].shape)
        del packed
        out_h = torch.empty(sess.out.shape, dtype=torch.float32).pin_memory()
        barrier(world)
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        # N > 1: every step ends with the north star's final gather, after
        # the decode path: the batch's outputs and C2 counts all-gathered
        # (ShardedSession.gather) and read back on rank 0
        gather = not args.no_gather and world > 1
        if gather:
            out_h = torch.empty(batch, hkv * group, d, dtype=torch.float32).pin_memory()
            cnt_h = torch.empty(batch, hkv * group, dtype=torch.int32).pin_memory()
        base = args.warmup + args.steps + gather_steps + prof_steps
        # Each step is what an autoregressive decode loop does: the step's
        # packed q | k_new | v_new goes in from pinned host memory and its
        # output must be back in host memory before the next step's query
        # exists -- so every step ends with a host wait on the output.  The
        # host wall clock (perf_counter) brackets all steps; the device
        # events give the same span on the GPU's clock.
        lat = []
        e0.record(cuda_stream)
        for t in range(base, base + e2e_steps):
            h0 = time.perf_counter()
            step_log.append(t % T_in)
            if not gather:
                # lfps_decode_step_host_io: the library copies the packed
                # inputs on its own stream beside the stats kernels and the
                # output back beside the commit kernel; the host waits for
                # the output only (lfps_wait_output) -- the commit may still
                # run while it builds the next step, which is stream-ordered
                # after it
                sess.decode_step_host(inh[t % T_in], frac, out_host=out_h)
                sess.wait_output()
            else:
                sess.decode_step_host(inh[t % T_in], frac)
                g_out, g_cnt, _ = ss.gather(with_c2=False)
                if rank == 0:
                    out_h.copy_(g_out, non_blocking=True)
                    cnt_h.copy_(g_cnt, non_blocking=True)
                cuda_stream.synchronize()        # the gathered output is in host memory
            lat.append(time.perf_counter() - h0)
        e1.record(cuda_stream)
        torch.cuda.synchronize(dev)
        e2e_ms = allmax(world, statistics.median(lat) * 1e3)
        dev_ms = e0.elapsed_time(e1) / e2e_steps
        sess.check_errors("e2e steps")
        d2h = out_h.numel() * 4 + (cnt_h.numel() * 4 if gather else 0)
        e2e = {"value": e2e_ms * 1e3, "unit": UNIT,
               "h2d_bytes_per_step": int(ind.numel() * ind.element_size()),
               "d2h_bytes_per_step": int(d2h if rank == 0 or not gather else 0),
               "timing": "median host wall-clock per step (perf_counter), each step waiting for "
                         "its output in pinned host memory before the next starts (lfps_wait_output; "
                         "the step's commit may still run); max over ranks",
               "device_span_us_per_step": dev_ms * 1e3,
               "api": ("ShardedSession: BatchedSession.decode_step_host on each rank's shard "
                       "(pinned host q|k_new|v_new in), then ShardedSession.gather: outputs and "
                       "C2 counts all-gathered, read back on rank 0" if gather else
                       "BatchedSession.decode_step_host = lfps_decode_step_host_io (pinned "
                       "packed q|k_new|v_new in, copied by the call beside the stats kernels; "
                       "the output copied to pinned host memory beside the commit kernel)")}

    # ---- recall vs the exact full-scan path, and its device time ----
    recall = None
    if recall_steps:
        etas, precs, ex_ms, errs_l, errs_x = [], [], [], [], []
        exact_kernel_ms = {}
        sess.exact_topk_step(stream.q[0], frac)        # warm-up (module load); read-only
        torch.cuda.synchronize(dev)
        base = args.warmup + args.steps + gather_steps + prof_steps + e2e_steps
        for t in range(base, base + recall_steps):
            torch.cuda.synchronize(dev)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            full = sess.full_attention(stream.q[t % T_in])       # N4: full attention
            a.record(cuda_stream)
            prof = t == base + recall_steps - 1
            if prof:
                _lib.profile_enable(True)
            sess.exact_topk_step(stream.q[t % T_in], frac)
            b.record(cuda_stream)
            if prof:
                torch.cuda.synchronize(dev)
                _lib.profile_enable(False)
                exact_kernel_ms = {k: v[1] / max(1, v[0]) for k, v in _lib.profile_collect().items()}
            ex_idx = sess.c2_idx.clone()
            ex_cnt = sess.counts.clone()
            ex_out = sess.out.clone()
            torch.cuda.synchronize(dev)
            ex_ms.append(a.elapsed_time(b))
            step(t)
            eta = sess.overlap(sess.c2_idx, sess.counts, ex_idx, ex_cnt)
            keep = sess.bypass == 0
            fn = full.double().norm(dim=-1).clamp_min(1e-12)
            errs_l.append(((sess.out.double() - full.double()).norm(dim=-1) / fn).flatten().cpu())
            errs_x.append(((ex_out.double() - full.double()).norm(dim=-1) / fn).flatten().cpu())
            etas.append(eta[keep].cpu().numpy())
            # precision: share of the LFPS selection inside the exact Top-k
            c2n = sess.counts[..., CNT_C2].double()
            exn = ex_cnt[..., CNT_C2].double()
            precs.append((eta * exn / c2n.clamp_min(1))[keep].cpu().numpy())
        eta_all = np.concatenate(etas)
        eta_sum = allsum(world, float(eta_all.sum()))
        eta_n = allsum(world, float(eta_all.size))
        prec = float(np.concatenate(precs).mean())
        recall = {"eta_mean": eta_sum / max(1.0, eta_n), "steps": recall_steps,
                  "precision_mean_rank0": prec,
                  "note": "eta = |C2 & I_exact| / k (attention.py:116-124); at 5% budget "
                          "|C2| = |probe| < k, so eta <= |probe| / k",
                  "exact_us_per_step": allmax(world, statistics.median(ex_ms[:-1] or ex_ms)) * 1e3,
                  "exact_kernel_ms": exact_kernel_ms,
                  "output_error_vs_full": {
                      "lfps_mean": float(torch.cat(errs_l).mean()),
                      "exact_topk_mean": float(torch.cat(errs_x).mean()),
                      "note": "relative L2 vs full softmax attention over every row "
                              "(full_attention_oracle / output_error, attention.py:88-134), "
                              "computed on the device"}}

    verified = None
    if args.verify and rank == 0 and not args.profile_only:
        verified = verify_units(sess, spec, stream, step_log, cfg, frac, args.verify, dev)
    if rank != 0:
        return
    cpu = None
    if not args.no_cpu and not args.profile_only and world == 1:
        cpu = cpu_leg(args.config, args.cpu_steps, 1, args.cpu_workers)
    value = ms * 1e3
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "dtypes": "fp64 tracker tables + gate, fp32 scores/softmax, bf16 K/V/q",
        "data": "synthetic (planted vertical bands + slash offsets; torch restatement of "
                "the reference generator synth.py)",
        "config": {"workload": desc, "batch": batch, "batch_per_gpu": b_local,
                   "shard_rank0": {"requests": [ss.shard.b0, ss.shard.nb],
                                   "kv_heads": [ss.shard.h0, ss.shard.nh]},
                   "context": ctx,
                   "q_heads": hkv * group, "kv_heads": hkv, "d": d, "topk_fraction": frac,
                   "sharding": ("(request, KV-head) units over ranks (sharded.plan_shards: requests "
                                "when B >= P, KV heads when B < P), no collective on the decode "
                                "path"),
                   "l2": "flushed before every timed step (512 MiB write); each step timed "
                         "by its own CUDA events",
                   "kv": ("paged (KvPool, %d MiB mapped)" % (sess.kv_mapped_bytes() >> 20)
                          if args.paged else "contiguous")},
        "gpu_launches": args.steps * _lib.load_library().lfps_decode_launches(
            C.byref(sess.dims), sess._params(frac).flags),
        "roofline": {"bound": "hbm", "kernel": dominant,
                     "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "traffic_source": "profiles/r02_ncu_traffic.json (ncu --set full, dram read+write "
                                       "per launch of this kernel at C4)" if traffic else None,
                     "algorithmic_bytes_per_launch": dom_bytes,
                     "avg_launch_ms": dom_ms, "peak_source": peak_src},
        "kernel_ms": kernel_ms,
        "kernels": per_kernel,
        "phase_us": phases,
        "kernel_algorithmic_bytes": {k: v for k, v in alg["kernels"].items() if k in kernel_ms},
        "step_algorithmic_bytes": int(alg["total"]),
        "step_achieved_GBps": alg["total"] / (ms * 1e-3) / 1e9,
        "reference_algorithm_bytes": int(alg["reference"]),
        "table_blocks_read_mean": alg["blocks_mean"],
        "clocks": clock_info,
        "setup_s": setup_s,
        "step_ms_min_max": [min(step_ms), max(step_ms)],
        "bypassed_sessions_last_step": bypass,
        "gate_near_epsilon_last_step": int(sess.gate_near_epsilon().sum()),
        "probe_mean": float(probe.mean()), "c2_mean": float(c2.mean()),
        "k_rows_distinct_per_unit": alg["k_rows_unit"], "v_rows_distinct_per_unit": alg["v_rows_unit"],
    }
    if verified:
        line["verified_units"] = verified
    if gather_ms is not None:
        line["step_with_gather_us"] = gather_ms * 1e3
        line["gather_note"] = ("device time per step incl. the all-gather of outputs [B, Hq, d] "
                               "and C2 counts over %s (value excludes it)" % dist_backend())
    if e2e:
        line["e2e"] = e2e
    if recall:
        line["recall"] = recall
        line["speedup_vs_exact_gpu"] = recall["exact_us_per_step"] / value
    if cpu:
        line["cpu_baseline"] = {"value": cpu["layer_step_us"], "unit": UNIT,
                                "cores": cpu["cores"], "kind": cpu["kind"],
                                "sample": cpu["sample"],
                                "cpu": cpu_model(),
                                "session_step_us_median": cpu["session_step_us_median"],
                                "exact_layer_step_us": cpu["exact_layer_step_us"]}
    print(json.dumps(line), flush=True)


def run_c3(args, world, rank, local):
    """BASELINE.json config 3: batch 16 x 128k context, all 32 layers of a
    decode step.  The 32 layers' K/V (8.6 GB each) do not all fit one B200
    next to their trackers, so one KV cache is shared by the 32 layer
    sessions (SURVEY.md §7 "Memory feasibility").  Everything else is per
    layer: each layer has its own query stream and last prefill queries
    (workload.gen_unit(layer=...): a layer-specific query walk and jitter
    over the shared planted keys), hence its own Eq. 4 tables, priors, probe
    sets and trajectory -- 32 distinct layers' work, only the K/V rows are
    shared (so the layers' row gathers can hit in L2 more than distinct
    caches would)."""
    import torch
    from paper_2506_15704_b200.config import LfpsConfig
    from paper_2506_15704_b200.session import BatchedSession
    from paper_2506_15704_b200.workload import GqaSpec, gen_unit, populate
    batch, ctx, layers, frac = 16, 131072, 32, 0.05
    b_local, b0 = shard_requests(batch, world, rank)
    T_in = 32
    cfg = LfpsConfig(d=128)
    dev = torch.device("cuda", torch.cuda.current_device())
    spec = GqaSpec(batch=b_local, kv_heads=8, group=4, d=128, n_prefill=ctx, steps=T_in,
                   seed=42 + 7919 * b0)
    n_max = ctx + args.warmup + args.steps + 8
    t_setup = time.time()
    sess = [BatchedSession(cfg, b_local, 8, 4, n_max=n_max, device=dev)]
    streams = [populate(sess[0], spec)]
    for layer in range(1, layers):
        s_l = BatchedSession(cfg, b_local, 8, 4, n_max=n_max, device=dev,
                             kv_cache=(sess[0].k_cache, sess[0].v_cache))
        s_l.n_ctx.copy_(sess[0].n_ctx)
        s_l.n_host = list(sess[0].n_host)
        q = torch.empty_like(streams[0].q)
        finals = torch.empty(b_local, 32, 128, dtype=torch.bfloat16, device=dev)
        for b in range(b_local):
            for h in range(8):
                u = gen_unit(spec, b, h, device=dev, layer=layer)
                s_l.bootstrap_tables((b * 8 + h) * 4, u.weights)
                q[:, b, h * 4:(h + 1) * 4] = u.queries.transpose(0, 1)
                finals[b, h * 4:(h + 1) * 4] = u.final_query
                del u
        s_l.bootstrap_stats(finals)
        torch.cuda.synchronize(dev)
        s_l.check_errors(f"bootstrap layer {layer}")
        sess.append(s_l)
        streams.append(type(streams[0])(q=q, k_new=streams[0].k_new, v_new=streams[0].v_new))
    for s_l in sess:
        s_l.split = not args.no_split
    setup_s = time.time() - t_setup

    side = torch.cuda.Stream(dev)
    pre_ev = [torch.cuda.Event() for _ in range(layers)]

    def token_step(t):
        i = t % T_in
        if not args.prefetch:
            for s_l, st in zip(sess, streams):
                s_l.decode_step(st.q[i], st.k_new[i], st.v_new[i], frac)
            return
        # The q-independent half of every layer's step (thresholds, C0, C1,
        # probe sets: lfps_decode_prefetch) runs ahead on a second stream,
        # in layer order, once the previous token's commits are done; the
        # layers' gate / finish / commit run in order on the main stream,
        # each after its own layer's prefetch (a real model's layer l + 1
        # queries exist only after layer l).
        main = torch.cuda.current_stream(dev)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            for s_l, ev in zip(sess, pre_ev):
                s_l.prefetch()
                ev.record(side)
        for s_l, st, ev in zip(sess, streams, pre_ev):
            main.wait_event(ev)
            s_l.decode_step(st.q[i], st.k_new[i], st.v_new[i], frac, prefetched=True)

    for t in range(args.warmup):
        token_step(t)
    torch.cuda.synchronize(dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier(world)
    torch.cuda.synchronize(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    for i in range(args.steps):
        flush.fill_(i & 255)
        evs[i][0].record()
        token_step(args.warmup + i)
        evs[i][1].record()
    torch.cuda.synchronize(dev)
    barrier(world)
    clock_info = clocks.stop()
    ms = allmax(world, sum(a.elapsed_time(b) for a, b in evs) / args.steps)
    for s_l in sess:
        s_l.check_errors("c3 steps")
    if rank != 0:
        return
    print(json.dumps({
        "metric": "LFPS index+sparse-attn us/decode-step (all 32 layers)", "value": ms * 1e3,
        "unit": "us/step", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong",
        "us_per_layer_step": ms * 1e3 / layers, "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic; one KV cache shared by the 32 layers, each layer with its own "
                 "query stream, prefill weights, tables and priors"),
        "config": {"workload": "C3: batch 16 x 128k context, 32 layers, Llama-3.1-8B shapes, "
                               "Top-k 5%", "batch": batch, "batch_per_gpu": b_local,
                   "context": ctx, "layers": layers, "topk_fraction": frac,
                   "l2": "flushed before every timed step",
                   "schedule": ("index ahead: every layer's candidate construction "
                                "(lfps_decode_prefetch) on a second stream, the layers' "
                                "gate/finish/commit in order on the main stream"
                                if args.prefetch else "layers in order, whole steps")},
        "clocks": clock_info, "setup_s": setup_s}), flush=True)


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    dist_init(world, local)
    if args.config == "c3":
        run_c3(args, world, rank, local)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
