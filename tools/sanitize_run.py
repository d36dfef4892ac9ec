"""Small end-to-end run for compute-sanitizer (memcheck / racecheck / synccheck):
decode steps through the per-session and the per-unit finish, a Top-k (1%)
step, and the exact path, on a B=1, 2 KV-head, G=4, n=2048 batch; then two
steps of a 256-session batch (8 x 8 KV heads x 4, d=64) through the
two-group stream split, the second with host inputs and output
(lfps_decode_step_host_io)."""
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
print("sanitize run ok")
