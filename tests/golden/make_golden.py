"""Generate tests/golden/sched_golden.json from the REFERENCE library.

Runs only where /root/reference exists (it is compiled from its own sources
into oracle/_ref/libfuseplan_ref.so by oracle/Makefile). The fixtures pin the
decision clock on the GPU box, where the reference is absent:
sample_lengths / make_batch outputs, simulate_serial / simulate_fused
timelines (sha256 of timeline_text plus key scalars), migration plans, sweep
curves and GAE vectors, for the reference's own fixtures (acceptance.cpp:371-390
"C7/C8" setup, test_genfuse.cpp cases) and this repo's workload configs.

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2409_13221_b200 import configs  # noqa: E402
from paper_2409_13221_b200.sched import (ClusterSpec, GenSimConfig, LengthDistribution, ModelSpec,  # noqa: E402
                                         Remaining, Sched)

REF_LIB = ROOT / "oracle" / "_ref" / "libfuseplan_ref.so"


def spec_7b():
    return ModelSpec("actor7b", 32, 32, 4096, 11008)


def spec_scorer(name):
    return ModelSpec(name, 16, 16, 2048, 8192)


def c7_setup():
    """acceptance.cpp:371-390 (sweep_setup / sweep_batch)."""
    cfg = GenSimConfig(actor=spec_7b(), num_instances=8, instance_gpus=8,
                       tasks=[("reward", spec_scorer("reward")), ("critic", spec_scorer("critic"))],
                       cluster=ClusterSpec(num_gpus=64, bs_max=256, kv_capacity_per_instance=24e9,
                                           interconnect_bandwidth=1e11))
    dist = LengthDistribution(median=200.0, p999_ratio=10.0, max_len=1024)
    return cfg, dist, 512, 256, 424242


def tiny():
    return ModelSpec("tiny", 4, 8, 256, 1024)


def base_config(num_instances, instance_gpus=1, bs_max=8, cap=0.0, bw=1e9):
    """test_genfuse.cpp:27-37."""
    return GenSimConfig(actor=tiny(), num_instances=num_instances, instance_gpus=instance_gpus,
                        tasks=[("reward", tiny())],
                        cluster=ClusterSpec(bs_max=bs_max, kv_capacity_per_instance=cap, interconnect_bandwidth=bw))


def digest(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def summarize(r):
    return {"gen_end": r.gen_end, "inf_end": r.inf_end, "total": r.total, "triggered": r.triggered,
            "plan": {"trigger_time": r.plan.trigger_time, "r_t": r.plan.r_t, "m": r.plan.m,
                     "destinations": r.plan.destinations, "mechanism": r.plan.mechanism,
                     "migrated": r.plan.migrated, "overhead": r.plan.overhead, "no_op": r.plan.no_op},
            "finish_sha": digest(json.dumps([repr(x) for x in r.finish_time])),
            "timeline_sha": digest(r.timeline), "n_events": len(r.events)}


def cases():
    """(name, batch-builder, cfg, r_t list) covering the reference fixtures and our workloads."""
    out = []
    cfg, dist, n, P, seed = c7_setup()
    out.append(("c7", ("lognormal", dict(median=dist.median, p999_ratio=dist.p999_ratio, max_len=dist.max_len), n, P, spec_7b().__dict__, seed), cfg,
                [0, 26, 51, 77, 102, 128, 154, 205, 256, 307, 358, 410, 461, 486]))
    out.append(("genfuse_sweep_grid", ("lognormal", dict(median=100.0, p999_ratio=10.0, max_len=1024), 64, 16,
                                       tiny().__dict__, 21), base_config(4, 2, bs_max=32), [6, 12, 19, 32, 44, 57]))
    out.append(("genfuse_kvcap", ("lognormal", dict(median=100.0, p999_ratio=10.0, max_len=512), 48, 16,
                                  tiny().__dict__, 33), None, [0, 8, 16, 32]))
    for name in ("toy", "gpt2s", "1.3b"):
        w = configs.WORKLOADS[name]
        for g in (2, 4, 8):
            lens = configs.zipf_lengths(w.n_prompts, w.max_new, w.zipf_s, w.zipf_lo, w.length_seed)
            gc = configs.gen_config(w, g, bs_max=256,
                                    kv_capacity=0.0 if name != "1.3b" else 40e9)
            out.append((f"{name}_g{g}", ("empirical", dict(max_len=w.max_new, empirical=lens), w.n_prompts,
                                          w.prompt_len, configs.model_spec("actor", w.actor).__dict__, 0), gc,
                        [0, round(0.1 * w.n_prompts), round(0.2 * w.n_prompts), round(0.3 * w.n_prompts)]))
    return out


def build_batch(s: Sched, spec):
    kind, dd, n, P, actor, seed = spec
    dist = LengthDistribution(kind=kind, **dd)
    return s.make_batch(dist, n, P, ModelSpec(**actor), seed)


def main():
    s = Sched(str(REF_LIB))
    gold = {"source": "reference library (oracle/_ref/libfuseplan_ref.so) built from /root/reference/proj/src",
            "cases": {}}
    for name, bspec, cfg, rts in cases():
        batch = build_batch(s, bspec)
        if cfg is None:  # KV-capped variant of test_genfuse.cpp:417-455
            kv_max = max(b.kv_bytes for b in batch)
            cfg = base_config(4, 2, bs_max=16, cap=8.0 * kv_max)
        entry = {"batch_spec": bspec, "targets_sha": digest(json.dumps([b.target_output_len for b in batch])),
                 "kv_sha": digest(json.dumps([repr(b.kv_bytes) for b in batch])),
                 "first_targets": [b.target_output_len for b in batch[:8]],
                 "sum_targets": sum(b.target_output_len for b in batch),
                 "serial": summarize(s.simulate_serial(batch, cfg)), "fused": {}}
        for r_t in rts:
            entry["fused"][str(r_t)] = summarize(s.simulate_fused(batch, cfg, r_t))
        sw = s.sweep_threshold(batch, cfg)
        entry["sweep"] = {"curve": sw.curve, "best_index": sw.best_index, "serial_total": sw.serial_total}
        gold["cases"][name] = (entry, cfg)
    # GAE vectors (numerics.cpp) on the reference's own fixtures + random rollouts
    import numpy as np
    rng = np.random.default_rng(99)
    gae = [{"rewards": [1.0, 1.0], "values": [0.0, 0.0, 0.0], "gamma": 0.9, "lam": 0.95},
           {"rewards": [2.0], "values": [1.0, 4.0], "gamma": 0.5, "lam": 0.7}]
    for _ in range(12):
        T = int(rng.integers(1, 600))
        gae.append({"rewards": list(rng.uniform(-10, 10, T)), "values": list(rng.uniform(-10, 10, T + 1)),
                    "gamma": float(rng.uniform(0, 1)), "lam": float(rng.uniform(0, 1))})
    for g in gae:
        g["recursive"] = list(s.gae_recursive(g["rewards"], g["values"], g["gamma"], g["lam"]))
        g["matrix"] = list(s.gae_matrix(g["rewards"], g["values"], g["gamma"], g["lam"]))
    gold["gae"] = gae
    # plan_migration KATs (test_genfuse.cpp:224-312)
    plans = []
    st = [Remaining(i, i % 8, 0.5e9, 5, 10, True) for i in range(256)]
    for bs, cap in ((128, 80e9), (512, 80e9), (100, 0.0)):
        cfg = base_config(8, bs_max=bs, cap=cap)
        plans.append(("ceilings", bs, cap, s.plan_migration(10.0, st, 256, cfg).__dict__))
    out_cases = {}
    for name, (entry, cfg) in gold["cases"].items():
        entry["cfg"] = json.loads(json.dumps(cfg, default=lambda o: o.__dict__))
        out_cases[name] = entry
    gold["cases"] = out_cases
    gold["plans"] = plans
    (Path(__file__).parent / "sched_golden.json").write_text(json.dumps(gold, indent=1))
    print("wrote", len(out_cases), "cases")


if __name__ == "__main__":
    main()
