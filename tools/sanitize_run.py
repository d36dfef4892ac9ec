"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
decode steps, a Top-k (1%) step, and the exact path, on a B=1, 2 KV-head,
G=4, n=2048 batch; two steps of a 256-session batch (8 x 8 KV heads x 4,
d=64) through the two-group stream split, the second with host inputs and
output (lfps_decode_step_host_io); two steps and the exact path over a
block-table KV cache; prefetched steps (lfps_decode_prefetch); and the
per-head fp64 stage API (k_stages.cu):
prefill_bootstrap, decode steps, topk_oracle, full attention."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from gpu_drive import Pair  # noqa: E402
from paper_2506_15704_b200.config import LfpsConfig  # noqa: E402
from paper_2506_15704_b200.workload import GqaSpec, gen_unit  # noqa: E402

spec = GqaSpec(batch=1, kv_heads=2, group=4, d=128, n_prefill=2048, steps=6, seed=1,
               slash_offsets=(64, 65), band_width=6)
units = [gen_unit(spec, 0, h) for h in range(2)]
K = np.stack([u.keys.float().numpy() for u in units])[None]
V = np.stack([u.values.float().numpy() for u in units])[None]
W = np.stack([u.weights.numpy() for u in units])[None]
F = np.stack([u.final_query.float().numpy() for u in units])[None]
Q = np.stack([u.queries.float().numpy() for u in units])[None]
pair = Pair(LfpsConfig(d=128), K, V, W, F, 2048)
for t in range(6):
    frac = 0.01 if t == 4 else 0.05
    res, outs = pair.step(Q[:, :, :, t], K[:, :, 2048 + t], V[:, :, 2048 + t], frac)
    pair.compare_step(res, outs)
import gpu_drive  # noqa: E402
qd = gpu_drive.bf16(Q[:, :, :, 0].reshape(1, -1, 128)).cuda()
pair.sess.exact_topk_step(qd, 0.05)
torch.cuda.synchronize()

spec = GqaSpec(batch=8, kv_heads=8, group=4, d=64, n_prefill=700, steps=2, seed=41,
               slash_offsets=(64, 65), band_width=6)
K, V, W, F, Q = [], [], [], [], []
for b in range(8):
    us = [gen_unit(spec, b, h) for h in range(8)]
    K.append([u.keys.float().numpy() for u in us])
    V.append([u.values.float().numpy() for u in us])
    W.append([u.weights.numpy() for u in us])
    F.append([u.final_query.float().numpy() for u in us])
    Q.append([u.queries.float().numpy() for u in us])
K, V, W, F, Q = (np.asarray(x) for x in (K, V, W, F, Q))
pair = Pair(LfpsConfig(d=64), K, V, W, F, 700)
pair.sess.split = True
for t in range(2):
    pair.host_io = t == 1           # lfps_decode_step_host_io: input copy beside stats
    res, outs = pair.step(Q[:, :, :, t], K[:, :, 700 + t], V[:, :, 700 + t], 0.05)
    pair.compare_step(res, outs, tables=(t == 1))
torch.cuda.synchronize()

# index ahead: lfps_decode_prefetch + LFPS_FLAG_PREFETCHED steps (split off, host I/O)
from gpu_drive import gqa_pair  # noqa: E402
pair, K, V, Q = gqa_pair(batch=2, kv_heads=2, n0=1500, steps=3, seed=61)
pair.prefetch = True
for t in range(3):
    pair.host_io = t == 2
    res, outs = pair.step(Q[:, :, :, t], K[:, :, 1500 + t], V[:, :, 1500 + t], 0.05)
    pair.compare_step(res, outs)
torch.cuda.synchronize()

# block-table KV (16-row blocks in a random order)
from gpu_drive import gqa_pair  # noqa: E402
pair, K, V, Q = gqa_pair(batch=2, kv_heads=2, n0=1500, steps=2, seed=59, block_rows=16)
for t in range(2):
    res, outs = pair.step(Q[:, :, :, t], K[:, :, 1500 + t], V[:, :, 1500 + t], 0.05)
    pair.compare_step(res, outs)
pair.sess.exact_topk_step(gpu_drive.bf16(Q[:, :, :, 1].reshape(2, -1, 128)).cuda(), 0.05)
torch.cuda.synchronize()

# the per-head stage API (fp64)
import paper_2506_15704_b200.lfps as lfps  # noqa: E402
rng = np.random.default_rng(3)
n, d, s_ = 300, 32, 4
cfg = lfps.LfpsConfig(d=d, s=s_, sink_count=2, local_window=3)
w = rng.random((s_, n - 2))
w /= w.sum(axis=1, keepdims=True)
ses = lfps.prefill_bootstrap(rng.standard_normal((n, d)), rng.standard_normal((n, d)), w,
                             rng.standard_normal(d), cfg)
for _ in range(4):
    lfps.decode_step(ses, rng.standard_normal(d), rng.standard_normal(d), rng.standard_normal(d),
                     0.05)
q = rng.standard_normal(d)
lfps.topk_oracle(q, ses.store, 15, 2)
lfps.full_attention_oracle(q, ses.store)
torch.cuda.synchronize()
print("sanitize run ok")
