"""Workload configurations of BASELINE.json and the synthetic length laws.

Model shapes (Llama-style: RMSNorm, RoPE, SwiGLU, GQA, untied head) for the
four north-star configs, and the bounded Zipf output-length
law P(k) ~ k^-s on [lo, max_len], drawn by inverse CDF from the reference's
splitmix64 Rng (proj/include/fuseplan/rng.hpp:10-44) and handed to the
scheduler as an empirical length list (genfuse.cpp:381-389), exactly as
SURVEY §7 hard-part 6 prescribes (the reference parser has no Zipf kind).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np

M64 = (1 << 64) - 1


@dataclass(frozen=True)
class Dims:
    num_layers: int
    hidden: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int

    def param_count(self, lm_head: bool = True) -> int:
        d, f, v = self.hidden, self.ffn, self.vocab
        qkv = (self.num_heads + 2 * self.num_kv_heads) * self.head_dim * d
        o = d * self.num_heads * self.head_dim
        per_layer = qkv + o + 3 * d * f
        return v * d + self.num_layers * per_layer + (v * d if lm_head else d)

    def kv_bytes_per_token(self) -> int:  # physical bf16 K + V
        return 2 * self.num_layers * self.num_kv_heads * self.head_dim * 2


@dataclass
class Workload:
    name: str
    actor: Dims
    ref: Dims
    critic: Dims
    reward: Dims
    n_prompts: int
    prompt_len: int
    max_new: int
    zipf_s: float = 1.0
    zipf_lo: int = 16
    gpus: tuple = (1,)
    length_seed: int = 424242


TOY = Dims(4, 256, 8, 8, 32, 1024, 2048)
GPT2S = Dims(12, 768, 12, 12, 64, 3072, 50257)
L13B = Dims(24, 2048, 16, 16, 128, 5632, 32000)
L8B = Dims(32, 4096, 32, 8, 128, 14336, 128256)

WORKLOADS = {
    "toy": Workload("toy", TOY, TOY, TOY, TOY, 64, 32, 512, zipf_s=1.0),
    "gpt2s": Workload("gpt2s", GPT2S, GPT2S, GPT2S, GPT2S, 512, 128, 1024, zipf_s=1.0),
    "1.3b": Workload("1.3b", L13B, L13B, L13B, L13B, 2048, 256, 1024, zipf_s=1.0, gpus=(2, 4, 8)),
    "8b": Workload("8b", L8B, L8B, L8B, L8B, 4096, 256, 4096, zipf_s=0.8, gpus=(8,)),
}


class Rng:
    """splitmix64 stream, bit-identical to fuseplan::Rng (rng.hpp:21-44)."""

    def __init__(self, seed: int):
        self.s = seed & M64

    def next_u64(self) -> int:
        self.s = (self.s + 0x9E3779B97F4A7C15) & M64
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


def zipf_lengths(n: int, max_len: int, s: float = 1.0, lo: int = 16, seed: int = 424242) -> list:
    """n lengths from P(k) ~ k^-s on [lo, max_len] (s = 0 is uniform)."""
    lo = min(lo, max_len)
    ks = np.arange(lo, max_len + 1, dtype=np.float64)
    w = ks ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    rng = Rng(seed)
    out = []
    for _ in range(n):
        u = rng.next_double()
        out.append(int(ks[min(int(np.searchsorted(cdf, u, side="right")), len(ks) - 1)]))
    return out


def model_spec(name: str, d: Dims):
    from .sched import ModelSpec
    return ModelSpec(name, d.num_layers, d.num_heads, d.hidden, d.ffn)


def calibration(w: Workload) -> dict | None:
    """CostModel constants fitted to measured B200 steps by tools/calibrate.py
    (profiles/r01_calibration_<workload>.json), or None."""
    import json
    from pathlib import Path
    p = Path(__file__).resolve().parent.parent / "profiles" / f"r01_calibration_{w.name}.json"
    return json.loads(p.read_text()) if p.exists() else None


def gen_config(w: Workload, instances: int, *, bs_max: int = 512, kv_capacity: float = 0.0,
               interconnect_bandwidth: float = 770e9, decode_step_base: float = 1e-3,
               time_per_token_coeff: float = 1e-12, calibrated: bool = False):
    """Decision-clock configuration (GenSimConfig) of a workload on `instances` B200s.

    instance_gpus = 1 (one engine per B200). The cost constants are the
    calibration knobs of SURVEY §8f row 1; calibrated=True takes them from the
    fit of measured B200 steps (tools/calibrate.py) when one exists.
    """
    from .sched import ClusterSpec, CostModel, GenSimConfig
    cal = calibration(w) if calibrated else None
    if cal:  # measured decode plateau / step base and forward cost
        bs_max, decode_step_base = int(cal["bs_max"]), float(cal["decode_step_base"])
        time_per_token_coeff = float(cal["time_per_token_coeff"])
    return GenSimConfig(
        actor=model_spec("actor", w.actor), num_instances=instances, instance_gpus=1,
        tasks=[("ref", model_spec("ref", w.ref)), ("reward", model_spec("reward", w.reward)),
               ("critic", model_spec("critic", w.critic))],
        cluster=ClusterSpec(num_gpus=instances, gpus_per_node=8, kv_capacity_per_instance=kv_capacity,
                            bs_max=bs_max, interconnect_bandwidth=interconnect_bandwidth),
        cost=CostModel(time_per_token_coeff=time_per_token_coeff, decode_step_base=decode_step_base))


def batch_for(w: Workload, sched, *, n: int | None = None, lengths: list | None = None, seed: int | None = None):
    """GenSample batch (ids 0..n-1) with Zipf lengths replayed as an empirical law."""
    from .sched import LengthDistribution
    n = n or w.n_prompts
    lens = lengths if lengths is not None else zipf_lengths(n, w.max_new, w.zipf_s, w.zipf_lo,
                                                            w.length_seed if seed is None else seed)
    dist = LengthDistribution(kind="empirical", max_len=w.max_new, empirical=list(lens))
    return sched.make_batch(dist, n, w.prompt_len, model_spec("actor", w.actor), 0)


def scaled(w: Workload, **kw) -> Workload:
    return replace(w, **kw)
