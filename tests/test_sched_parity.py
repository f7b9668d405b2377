"""Decision clock parity: the product scheduler (C++ in csrc/host, through the
C ABI of include/fp_sched.h) against the reference implementation.

* golden fixtures (tests/golden/sched_golden.json, generated from the
  reference library by tests/golden/make_golden.py) — runs everywhere;
* live differential fuzzing against oracle/_ref/libfuseplan_ref.so (the
  reference sources compiled from /root/reference) — where it is built.
Bit-exact: every float is compared with ==, timelines by their full text.
"""
import hashlib
import json
import random
from pathlib import Path

import numpy as np
import pytest

from paper_2409_13221_b200 import _lib
from paper_2409_13221_b200.sched import (ClusterSpec, CostModel, GenSample, GenSimConfig, LengthDistribution,
                                         ModelSpec, Remaining)

GOLD = json.loads((Path(__file__).parent / "golden" / "sched_golden.json").read_text())


def digest(text):
    return hashlib.sha256(text.encode()).hexdigest()


def cfg_from(d):
    return GenSimConfig(actor=ModelSpec(**d["actor"]), num_instances=d["num_instances"],
                        instance_gpus=d["instance_gpus"], tasks=[(n, ModelSpec(**m)) for n, m in d["tasks"]],
                        cluster=ClusterSpec(**d["cluster"]), cost=CostModel(**d["cost"]))


def batch_from(s, spec):
    kind, dd, n, P, actor, seed = spec
    return s.make_batch(LengthDistribution(kind=kind, **dd), n, P, ModelSpec(**actor), seed)


def summarize(r):
    return {"gen_end": r.gen_end, "inf_end": r.inf_end, "total": r.total, "triggered": r.triggered,
            "plan": {"trigger_time": r.plan.trigger_time, "r_t": r.plan.r_t, "m": r.plan.m,
                     "destinations": r.plan.destinations, "mechanism": r.plan.mechanism,
                     "migrated": r.plan.migrated, "overhead": r.plan.overhead, "no_op": r.plan.no_op},
            "finish_sha": digest(json.dumps([repr(x) for x in r.finish_time])),
            "timeline_sha": digest(r.timeline), "n_events": len(r.events)}


@pytest.mark.parametrize("name", sorted(GOLD["cases"]))
def test_golden_case(sched, name):
    g = GOLD["cases"][name]
    cfg = cfg_from(g["cfg"])
    batch = batch_from(sched, g["batch_spec"])
    assert digest(json.dumps([b.target_output_len for b in batch])) == g["targets_sha"]
    assert digest(json.dumps([repr(b.kv_bytes) for b in batch])) == g["kv_sha"]
    assert summarize(sched.simulate_serial(batch, cfg)) == g["serial"]
    for r_t, want in g["fused"].items():
        assert summarize(sched.simulate_fused(batch, cfg, int(r_t))) == want, r_t
    sw = sched.sweep_threshold(batch, cfg)
    assert [list(p) for p in sw.curve] == g["sweep"]["curve"]
    assert sw.best_index == g["sweep"]["best_index"] and sw.serial_total == g["sweep"]["serial_total"]


def test_c7_acceptance_bands(sched):
    """acceptance.cpp:392-432 (C7 interior argmin in [0.10, 0.35], fused <= serial/1.1; C8 preservation)."""
    g = GOLD["cases"]["c7"]
    cfg = cfg_from(g["cfg"])
    batch = batch_from(sched, g["batch_spec"])
    assert g["first_targets"] == [188, 119, 94, 68, 101, 143, 112, 233] and g["sum_targets"] == 129834
    sw = sched.sweep_threshold(batch, cfg)
    best = sw.curve[sw.best_index]
    assert 0 < sw.best_index < len(sw.curve) - 1
    assert 0.10 <= best[0] <= 0.35 and best[2] <= sw.serial_total / 1.1
    serial = sched.simulate_serial(batch, cfg)
    for pct in range(5, 100, 5):
        r_t = int(round(pct / 100 * len(batch) + 1e-12))
        f = sched.simulate_fused(batch, cfg, r_t)
        slack = 1e-9 * serial.gen_end
        assert all(ff <= sf + f.plan.overhead + slack for ff, sf in zip(f.finish_time, serial.finish_time))


def test_gae_golden(sched):
    for g in GOLD["gae"]:
        rec = sched.gae_recursive(g["rewards"], g["values"], g["gamma"], g["lam"])
        mat = sched.gae_matrix(g["rewards"], g["values"], g["gamma"], g["lam"])
        assert list(rec) == g["recursive"] and list(mat) == g["matrix"]
    a = sched.gae_recursive([1.0, 1.0], [0.0, 0.0, 0.0], 0.9, 0.95)
    assert abs(a[0] - 1.855) <= 1e-12 and a[1] == 1.0  # test_numerics.cpp:35-49


def test_plan_kats(sched):
    """test_genfuse.cpp:224-312 literal expectations."""
    tiny = ModelSpec("tiny", 4, 8, 256, 1024)

    def base(n, bs, cap=0.0, bw=1e9):
        return GenSimConfig(actor=tiny, num_instances=n, instance_gpus=1, tasks=[("reward", tiny)],
                            cluster=ClusterSpec(bs_max=bs, kv_capacity_per_instance=cap, interconnect_bandwidth=bw))
    st = [Remaining(i, i % 8, 0.5e9, 5, 10, True) for i in range(256)]
    assert sched.plan_migration(10.0, st, 256, base(8, 128, 80e9)).m == 2
    assert sched.plan_migration(10.0, st, 256, base(8, 512, 80e9)).m == 2
    assert sched.plan_migration(10.0, st, 256, base(8, 100)).m == 3
    st, i = [], 0
    for ins, c in enumerate([30, 5, 4, 1]):
        for _ in range(c):
            st.append(Remaining(i, ins, 1.0, 0, 8, True))
            i += 1
    p = sched.plan_migration(1.0, st, 40, base(4, 20))
    assert p.m == 2 and p.destinations == [0, 1] and len(p.migrated) == 5
    tied = [Remaining(0, 3, 1.0, 0, 8, True), Remaining(1, 1, 1.0, 0, 8, True)]
    assert sched.plan_migration(0.0, tied, 40, base(4, 20)).destinations == [1, 3]
    st = [Remaining(0, 0, 4e6, 100, 32, True), Remaining(1, 1, 6e6, 50, 32, True), Remaining(2, 1, 2e6, 10, 32, False)]
    fast = sched.plan_migration(0.0, st, 2, base(4, 64, bw=1e11))
    assert fast.m == 1 and fast.destinations == [1] and fast.migrated == [0]
    assert fast.mechanism == "kv_transfer" and fast.overhead == pytest.approx(4e6 / 1e11)
    slow = sched.plan_migration(0.0, st, 2, base(4, 64, bw=1e6))
    assert slow.mechanism == "recompute_prefill"
    for n, bs, r_t, ss in ((2, 2, 8, [Remaining(i, i % 2, 1.0, 0, 8, True) for i in range(8)]),
                           (2, 2, 0, [Remaining(0, 0, 1.0, 0, 8, True)]), (2, 2, 4, [])):
        assert sched.plan_migration(0.0, ss, r_t, base(n, bs)).no_op


def test_hand_checked_migration(sched):
    """test_genfuse.cpp:329-375: trigger 0.02, m=1, dest {0}, migrated {5, 6}."""
    tiny = ModelSpec("tiny", 4, 8, 256, 1024)
    cfg = GenSimConfig(actor=tiny, num_instances=4, instance_gpus=1, tasks=[("reward", tiny)],
                       cluster=ClusterSpec(bs_max=8, interconnect_bandwidth=1e9))
    batch = [GenSample(i, 0, t, 0, 1.0) for i, t in enumerate([1, 1, 1, 1, 20, 30, 40, 2])]
    serial = sched.simulate_serial(batch, cfg)
    assert serial.gen_end == pytest.approx(0.40, rel=1e-12)
    f = sched.simulate_fused(batch, cfg, 4)
    assert f.triggered and not f.plan.no_op
    assert f.plan.trigger_time == pytest.approx(0.02, rel=1e-9) and f.plan.m == 1
    assert f.plan.destinations == [0] and f.plan.migrated == [5, 6] and f.plan.mechanism == "kv_transfer"
    outs = [(e[1], e[3]) for e in f.events if e[2] == "migrate_out"]
    assert sorted(outs) == [(1, 5), (2, 6)]
    assert f.total < serial.total


def test_error_statuses(sched):
    tiny = ModelSpec("tiny", 4, 8, 256, 1024)
    cfg = GenSimConfig(actor=tiny, num_instances=1, instance_gpus=1, tasks=[("reward", tiny)],
                       cluster=ClusterSpec(bs_max=8, kv_capacity_per_instance=0.5))
    with pytest.raises(_lib.InfeasibleError):
        sched.simulate_serial([GenSample(0, 0, 1, 0, 1.0), GenSample(1, 0, 2, 0, 1.0)], cfg)
    cfg.cluster.bs_max = 0
    with pytest.raises(_lib.ConfigError):
        sched.simulate_serial([GenSample(0, 0, 1, 0, 1.0)], cfg)
    with pytest.raises(_lib.ConfigError):
        sched.sample_lengths(LengthDistribution(p999_ratio=1.0), 10, 0)
    with pytest.raises(_lib.ConfigError):
        sched.sample_lengths(LengthDistribution(kind="empirical", empirical=[]), 5, 0)
    assert sched.sample_lengths(LengthDistribution(kind="empirical", empirical=[5, 900, 3], max_len=100), 5, 42) == \
        [5, 100, 3, 5, 100]
    with pytest.raises(_lib.ConfigError):
        sched.load_length_file("/nonexistent/lengths.txt")
    with pytest.raises(_lib.ConfigError):
        sched.gae_recursive([1.0], [0.0], 0.9, 0.9)


def test_length_file(sched, tmp_path):
    p = tmp_path / "l.txt"
    p.write_text("12\n\n  7 \n3000\n")
    assert sched.load_length_file(str(p)) == [12, 7, 3000]
    p.write_text("12\nnope\n")
    with pytest.raises(_lib.ConfigError):
        sched.load_length_file(str(p))


def _random_case(rng: random.Random):
    tiny = ModelSpec("m", rng.choice([2, 4, 8]), 4, 256, 512)
    n_inst = rng.randint(1, 8)
    dist = LengthDistribution(median=rng.uniform(20, 200), p999_ratio=rng.uniform(1.5, 20),
                              max_len=rng.choice([64, 256, 1024]))
    n = rng.randint(1, 200)
    prompt = rng.choice([0, 1, 16, 128])
    cap = rng.choice([0.0, 0.0, 1.0]) * rng.uniform(1, 40) * (prompt + dist.max_len) * 4 * 2 * 256
    cfg = GenSimConfig(actor=tiny, num_instances=n_inst, instance_gpus=rng.choice([1, 2, 8]),
                       tasks=[("ref", tiny), ("critic", ModelSpec("c", 2, 4, 128, 256))],
                       cluster=ClusterSpec(bs_max=rng.choice([1, 4, 16, 64, 256]), kv_capacity_per_instance=cap,
                                           interconnect_bandwidth=rng.choice([1e3, 1e6, 1e9, 1e12])),
                       cost=CostModel(decode_step_base=rng.choice([0.0, 1e-3, 0.01]),
                                      time_per_token_coeff=rng.choice([1e-15, 1e-12, 1e-9])))
    return dist, n, prompt, tiny, cfg, rng.randint(0, 1 << 40)


@pytest.mark.parametrize("seed", range(40))
def test_differential_vs_reference_library(sched, ref_sched, seed):
    rng = random.Random(seed)
    dist, n, prompt, actor, cfg, s = _random_case(rng)
    b1 = sched.make_batch(dist, n, prompt, actor, s)
    b2 = ref_sched.make_batch(dist, n, prompt, actor, s)
    assert b1 == b2
    try:
        r2 = ref_sched.simulate_serial(b2, cfg)
    except _lib.FpError as e:
        with pytest.raises(type(e)):
            sched.simulate_serial(b1, cfg)
        return
    assert sched.simulate_serial(b1, cfg) == r2
    for r_t in sorted({0, 1, n // 10, n // 5, n // 3, n // 2, n, n + 3}):
        assert sched.simulate_fused(b1, cfg, r_t) == ref_sched.simulate_fused(b2, cfg, r_t), r_t
    assert sched.sweep_threshold(b1, cfg) == ref_sched.sweep_threshold(b2, cfg)


@pytest.mark.parametrize("seed", range(10))
def test_differential_plan_migration(sched, ref_sched, seed):
    rng = random.Random(1000 + seed)
    n_inst = rng.randint(1, 8)
    tiny = ModelSpec("m", 4, 4, 256, 512)
    st = [Remaining(i, rng.randrange(n_inst), rng.uniform(1e5, 1e9), rng.randint(0, 500), rng.randint(0, 300),
                    rng.random() < 0.7) for i in range(rng.randint(0, 300))]
    for r_t in (0, 1, 5, 50, 300):
        cfg = GenSimConfig(actor=tiny, num_instances=n_inst, instance_gpus=rng.choice([1, 4]), tasks=[],
                           cluster=ClusterSpec(bs_max=rng.choice([1, 8, 64]),
                                               kv_capacity_per_instance=rng.choice([0.0, 1e10, 8e10]),
                                               interconnect_bandwidth=rng.choice([1e6, 1e9, 1e12])))
        assert sched.plan_migration(3.5, st, r_t, cfg) == ref_sched.plan_migration(3.5, st, r_t, cfg)


def test_gae_random_vs_reference(sched, ref_sched):
    rng = np.random.default_rng(7)
    for _ in range(50):
        T = int(rng.integers(1, 2000))
        r, v = rng.uniform(-10, 10, T), rng.uniform(-10, 10, T + 1)
        g, l = float(rng.uniform(0, 1)), float(rng.uniform(0, 1))
        assert np.array_equal(sched.gae_recursive(r, v, g, l), ref_sched.gae_recursive(r, v, g, l))
        assert np.array_equal(sched.gae_matrix(r, v, g, l), ref_sched.gae_matrix(r, v, g, l))
