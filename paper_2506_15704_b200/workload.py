"""Synthetic GQA decode workloads with planted vertical/slash structure.

Harness input, not part of the decode path.  Restates the recipe of the
reference generator (pkg/src/lfps/synth.py:112-208) in torch so it runs at
the survey's configs (B up to 64, 128k context) on the device, and extends
it to GQA: every (request, KV-head) unit owns one K/V row store shared by its
G query heads, and each query head plants its own vertical bands and slash
offsets into the shared rows (SURVEY.md §8(d) "Synthetic inputs").

Recipe per unit (synth.py line refs in brackets):
* keys  = noise_scale * N(0, 1) rows (key_correlation 0 -> i.i.d.) [400]
* values = N(0, 1) rows [401]
* one orthonormal direction per (q-head, band); noise is projected out of
  those directions in keys and queries, then every band member key gets
  amp * u with amp = sqrt(signal_gain * sqrt(d)) [403-424]
* queries follow an AR(1) walk (query_correlation) [415]; each carries
  amp * u for its own bands, a roaming spotlight near each band edge and
  point boosts that lift the score of position t - o by signal_gain for its
  slash offsets o (jittered) [432-461]; optional sink boosts [462-464]
* prefill weights: exact softmax of the trailing s prefill queries over
  rows [0, t], non-sink part renormalised [467-479]

All tensors leave as bf16 (K, V, q) plus fp32 prefill weights.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch


@dataclass(frozen=True)
class GqaSpec:
    batch: int = 1
    kv_heads: int = 8
    group: int = 4
    d: int = 128
    n_prefill: int = 16384
    steps: int = 64
    s: int = 32
    sink_count: int = 4
    signal_gain: float = 5.0
    noise_scale: float = 0.5
    query_correlation: float = 0.999
    band_width: int = -1          # -1: about n/650
    band_fracs: tuple = (0.13, 0.40, 0.75)
    slash_offsets: tuple = (-1, -1)  # -1: (128,129) at <= 8k else (300,301)
    plant_jitter: int = 2
    sink_gain: float = 0.0
    sink_heads: tuple = ()        # q-head indices (within a request) that get sink_gain
    seed: int = 42
    extra_rows: int = 0           # capacity headroom beyond n_prefill + steps

    @property
    def q_heads(self) -> int:
        return self.kv_heads * self.group

    @property
    def width(self) -> int:
        if self.band_width >= 0:
            return self.band_width
        return max(2, self.n_prefill // 650)

    @property
    def offsets(self) -> tuple:
        if self.slash_offsets != (-1, -1):
            return tuple(self.slash_offsets)
        return (128, 129) if self.n_prefill <= 8192 else (300, 301)


@dataclass
class GqaUnitData:
    """One unit's inputs (all on ``device``)."""

    keys: torch.Tensor        # [n_total, d] bf16
    values: torch.Tensor      # [n_total, d] bf16
    queries: torch.Tensor     # [G, steps, d] bf16
    final_query: torch.Tensor  # [G, d] bf16 (last prefill query)
    weights: torch.Tensor | None = None   # [G, s, n_prefill - S] fp32


def _unit_generator(spec: GqaSpec, b: int, h: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(spec.seed * 1_000_003 + b * 1009 + h)
    return g


def gen_unit(spec: GqaSpec, b: int, h: int, device="cpu", with_weights=True,
             layer: int = 0) -> GqaUnitData:
    """Generate one (request b, KV-head h) unit.

    ``layer`` > 0 gives another attention layer over the SAME K/V rows (the
    keys, values and planted band directions are layer 0's): its query walk
    and jitter come from a layer-specific generator, so its queries, prefill
    weights (hence tables) and trajectory differ (bench.py C3)."""
    d, G, S = spec.d, spec.group, spec.sink_count
    n0, steps = spec.n_prefill, spec.steps
    total = n0 + steps
    gen = _unit_generator(spec, b, h, device)
    f32 = torch.float32
    keys = spec.noise_scale * torch.randn(total, d, generator=gen, device=device, dtype=f32)
    values = torch.randn(total, d, generator=gen, device=device, dtype=f32)
    scale = math.sqrt(d)
    w = spec.width
    nb = len(spec.band_fracs)
    # per-head band centres: the head's own shift keeps heads distinct
    centres = []
    for g in range(G):
        row = []
        for j, fr in enumerate(spec.band_fracs):
            c = int(fr * n0) + (g * 37 + j * 11) % max(1, n0 // 50)
            row.append(min(max(c, S + w), n0 - w - 1))
        centres.append(row)
    nq = spec.s + steps
    first_q = n0 - spec.s
    # AR(1) query walk per head
    base = torch.randn(G, nq, d, generator=gen, device=device, dtype=f32)
    qgen = gen
    if layer:
        qgen = torch.Generator(device=device)
        qgen.manual_seed(spec.seed * 1_000_003 + b * 1009 + h + 7_919_000 * layer)
        base = torch.randn(G, nq, d, generator=qgen, device=device, dtype=f32)
    rho = spec.query_correlation
    blend = math.sqrt(1.0 - rho * rho)
    walk = torch.empty_like(base)
    walk[:, 0] = base[:, 0]
    for i in range(1, nq):
        walk[:, i] = rho * walk[:, i - 1] + blend * base[:, i]
    q = spec.noise_scale * walk
    amp = math.sqrt(spec.signal_gain * scale) if spec.signal_gain > 0 else 0.0
    if amp > 0 and d > G * nb:
        raw = torch.randn(d, G * nb, generator=gen, device=device, dtype=f32)
        dirs, _ = torch.linalg.qr(raw)
        dirs = dirs.T.contiguous()                       # [G*nb, d]
        keys -= (keys @ dirs.T) @ dirs
        q -= (q @ dirs.T) @ dirs
        for g in range(G):
            for j in range(nb):
                u = dirs[g * nb + j]
                c = centres[g][j]
                keys[c - w: c + w + 1] += amp * u
                q[g] += amp * u
    knorm = keys.norm(dim=1).clamp_min(1e-30)
    kdir = keys / knorm[:, None]
    jit = spec.plant_jitter
    t_idx = torch.arange(first_q, total, device=device)

    def boost(g, pos, lift):
        # lift q[g, i] . K[pos_i] / sqrt(d) by exactly `lift` (synth.py:432-434)
        q[g] += (lift * scale / knorm[pos])[:, None] * kdir[pos]

    if amp > 0:
        for g in range(G):
            if jit:
                for j in range(nb):
                    side = torch.where(torch.rand(nq, generator=qgen, device=device) < 0.5, 1, -1)
                    mag = torch.randint(max(0, w - 1), w + jit + 1, (nq,), generator=qgen,
                                        device=device)
                    pos = (centres[g][j] + side * mag).clamp(min=S)
                    pos = torch.minimum(pos, t_idx)
                    boost(g, pos, spec.signal_gain)
            for o in spec.offsets:
                dj = torch.randint(-jit, jit + 1, (nq,), generator=qgen, device=device) if jit \
                    else torch.zeros(nq, dtype=torch.long, device=device)
                pos = (t_idx - o + dj).clamp(min=S)
                pos = torch.minimum(pos, t_idx)
                boost(g, pos, spec.signal_gain)
    if spec.sink_gain > 0:
        for g in range(G):
            if (h * G + g) in spec.sink_heads or not spec.sink_heads:
                gain = spec.sink_gain * (g + 1) / G
                for j in range(S):
                    boost(g, torch.full((nq,), j, device=device, dtype=torch.long), gain)
    kb = keys.to(torch.bfloat16)
    vb = values.to(torch.bfloat16)
    qb = q.to(torch.bfloat16)
    unit = GqaUnitData(keys=kb, values=vb, queries=qb[:, spec.s:].contiguous(),
                       final_query=qb[:, spec.s - 1].contiguous())
    if with_weights:
        unit.weights = prefill_weights(kb[:n0], qb[:, : spec.s], S)
    return unit


def prefill_weights(keys_bf16: torch.Tensor, prefill_q_bf16: torch.Tensor, sink: int) -> torch.Tensor:
    """Exact causal softmax weights of the trailing s prefill queries, non-sink
    range renormalised, zero beyond each step's causal extent (synth.py:467-479).

    keys_bf16 [n0, d]; prefill_q_bf16 [G, s, d] (query c sits at t = n0 - s + c)."""
    n0, d = keys_bf16.shape
    G, s, _ = prefill_q_bf16.shape
    k = keys_bf16.float()
    qf = prefill_q_bf16.float()
    logits = torch.einsum("gsd,nd->gsn", qf, k) / math.sqrt(d)     # [G, s, n0]
    t = torch.arange(n0 - s, n0, device=k.device)
    cols = torch.arange(n0, device=k.device)
    mask = cols[None, :] > t[:, None]                                # beyond causal extent
    logits = logits.masked_fill(mask[None], float("-inf"))
    w = torch.softmax(logits.double(), dim=-1)[..., sink:]
    w = w / w.sum(dim=-1, keepdim=True)
    return w.float().contiguous()


def bf16_to_f64(x: torch.Tensor):
    """Host fp64 numpy copy of a bf16 tensor (exact upcast)."""
    return x.detach().to("cpu", torch.float64).numpy()


@dataclass
class StepStream:
    """Per-step decode inputs for a whole batch, resident on the device."""

    q: torch.Tensor       # bf16 [T, B, Hq, d]
    k_new: torch.Tensor   # bf16 [T, B, Hkv, d]
    v_new: torch.Tensor   # bf16 [T, B, Hkv, d]


def populate(session, spec: GqaSpec, progress=None) -> StepStream:
    """Fill a BatchedSession with the spec's synthetic prefill (KV rows,
    Eq. 4 tables, gate priors) and return the decode-step inputs.  Runs
    unit by unit on the session's device so 128k x 64 fits in memory."""
    dev = session.device
    B, Hkv, G, d = spec.batch, spec.kv_heads, spec.group, spec.d
    n0, T = spec.n_prefill, spec.steps
    q = torch.empty(T, B, Hkv * G, d, dtype=torch.bfloat16, device=dev)
    kn = torch.empty(T, B, Hkv, d, dtype=torch.bfloat16, device=dev)
    vn = torch.empty(T, B, Hkv, d, dtype=torch.bfloat16, device=dev)
    finals = torch.empty(B, Hkv * G, d, dtype=torch.bfloat16, device=dev)
    for b in range(B):
        for h in range(Hkv):
            u = gen_unit(spec, b, h, device=dev)
            session.load_unit(b, h, u.keys[:n0], u.values[:n0])
            s0 = b * Hkv * G + h * G
            session.bootstrap_tables(s0, u.weights)
            q[:, b, h * G:(h + 1) * G] = u.queries.transpose(0, 1)
            kn[:, b, h] = u.keys[n0:n0 + T]
            vn[:, b, h] = u.values[n0:n0 + T]
            finals[b, h * G:(h + 1) * G] = u.final_query
            del u
        if progress:
            progress(b)
    session.bootstrap_stats(finals)
    torch.cuda.synchronize(dev)
    session.check_errors("bootstrap")
    return StepStream(q=q, k_new=kn, v_new=vn)
