"""Python mirror of the reference's gen+inf scheduler API (genfuse.hpp / numerics.hpp).

Every function calls through the C ABI of include/fp_sched.h; `Sched(lib)`
binds to the product library by default, or to any library exporting the same
ABI — notably oracle/_ref/libfuseplan_ref.so, the reference sources built
from /root/reference, which is how tests/test_sched_parity.py diffs the two.

Names and argument meaning follow proj/include/fuseplan/genfuse.hpp:15-141:
LengthDistribution, sample_lengths, load_length_file, make_batch, GenSimConfig,
plan_migration, simulate_serial, simulate_fused, sweep_threshold,
timeline_text; plus gae_recursive / gae_matrix (numerics.hpp:18-25).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import check


@dataclass
class ModelSpec:
    name: str
    num_layers: int
    num_heads: int
    hidden_size: int
    intermediate_size: int

    def c(self, keep: list) -> _lib.ModelSpec:
        b = self.name.encode()
        keep.append(b)
        return _lib.ModelSpec(b, self.num_layers, self.num_heads, self.hidden_size, self.intermediate_size)


@dataclass
class CostModel:
    time_per_token_coeff: float = 1e-12
    backward_forward_ratio: float = 2.0
    activation_bytes_coeff: float = 1.0
    decode_step_base: float = 0.01
    comm_bandwidth: float = 1e9


@dataclass
class ClusterSpec:
    num_gpus: int = 0
    gpus_per_node: int = 8
    activation_capacity_per_stage: float = 0.0
    kv_capacity_per_instance: float = 0.0
    bs_max: int = 1
    interconnect_bandwidth: float = 1e9


@dataclass
class GenSimConfig:
    actor: ModelSpec
    num_instances: int = 8
    instance_gpus: int = 8
    tasks: list = field(default_factory=list)  # [(name, ModelSpec)]
    cluster: ClusterSpec = field(default_factory=ClusterSpec)
    cost: CostModel = field(default_factory=CostModel)

    def c(self, keep: list) -> _lib.GenConfig:
        n = len(self.tasks)
        specs = (_lib.ModelSpec * max(n, 1))()
        names = (C.c_char_p * max(n, 1))()
        for i, (nm, spec) in enumerate(self.tasks):
            specs[i] = spec.c(keep)
            b = nm.encode()
            keep.append(b)
            names[i] = b
        keep += [specs, names]
        cl = _lib.ClusterSpec(self.cluster.num_gpus, self.cluster.gpus_per_node,
                              self.cluster.activation_capacity_per_stage, self.cluster.kv_capacity_per_instance,
                              self.cluster.bs_max, self.cluster.interconnect_bandwidth)
        co = _lib.CostModel(self.cost.time_per_token_coeff, self.cost.backward_forward_ratio,
                            self.cost.activation_bytes_coeff, self.cost.decode_step_base, self.cost.comm_bandwidth)
        return _lib.GenConfig(self.actor.c(keep), self.num_instances, self.instance_gpus, n, specs, names, cl, co)


@dataclass
class LengthDistribution:
    kind: str = "lognormal"  # or "empirical"
    median: float = 200.0
    p999_ratio: float = 10.0
    max_len: int = 1024
    empirical: list = field(default_factory=list)

    def c(self, keep: list) -> _lib.LengthDist:
        arr = (C.c_int32 * max(len(self.empirical), 1))(*self.empirical)
        keep.append(arr)
        return _lib.LengthDist(1 if self.kind == "empirical" else 0, self.median, self.p999_ratio, self.max_len,
                               arr, len(self.empirical))


@dataclass
class GenSample:
    id: int
    prompt_len: int
    target_output_len: int
    generated: int = 0
    kv_bytes: float = 0.0


@dataclass
class Remaining:
    id: int
    instance: int
    kv_bytes: float
    generated: int
    prompt_len: int
    admitted: bool


@dataclass
class MigrationPlan:
    trigger_time: float
    r_t: int
    m: int
    destinations: list
    mechanism: str  # "kv_transfer" | "recompute_prefill"
    migrated: list
    overhead: float
    no_op: bool


@dataclass
class GenStageResult:
    gen_end: float
    inf_end: float
    total: float
    plan: MigrationPlan
    triggered: bool
    finish_time: list
    events: list  # (time, instance, kind, sample)
    timeline: str


@dataclass
class SweepResult:
    curve: list  # (ratio, r_t, fused_total)
    best_index: int
    serial_total: float


def batch_to_c(batch, keep: list):
    arr = (_lib.GenSample * max(len(batch), 1))()
    for i, s in enumerate(batch):
        arr[i] = _lib.GenSample(s.id, s.prompt_len, s.target_output_len, s.generated, s.kv_bytes)
    keep.append(arr)
    return arr


def _plan_from(info: _lib.PlanInfo, dests, migrated) -> MigrationPlan:
    return MigrationPlan(info.trigger_time, info.r_t, info.m, list(dests), "kv_transfer" if info.mechanism == 0
                         else "recompute_prefill", list(migrated), info.overhead, bool(info.no_op))


class Sched:
    """The gen+inf scheduler API over one C library (product or oracle)."""

    def __init__(self, lib: C.CDLL | str | None = None):
        self.lib = lib if isinstance(lib, C.CDLL) else _lib.load(lib, engine=False if lib else None)

    # --- lengths / batch -------------------------------------------------------------------
    def sample_lengths(self, dist: LengthDistribution, n: int, seed: int) -> list:
        keep: list = []
        out = (C.c_int32 * max(n, 1))()
        check(self.lib, self.lib.fp_sample_lengths(C.byref(dist.c(keep)), n, seed, out))
        return list(out[:n])

    def load_length_file(self, path: str) -> list:
        cnt = C.c_int32(0)
        check(self.lib, self.lib.fp_load_length_file(path.encode(), None, 0, C.byref(cnt)))
        out = (C.c_int32 * max(cnt.value, 1))()
        check(self.lib, self.lib.fp_load_length_file(path.encode(), out, cnt.value, C.byref(cnt)))
        return list(out[:cnt.value])

    def make_batch(self, dist: LengthDistribution, n: int, prompt_len: int, actor: ModelSpec, seed: int) -> list:
        keep: list = []
        out = (_lib.GenSample * max(n, 1))()
        check(self.lib, self.lib.fp_make_batch(C.byref(dist.c(keep)), n, prompt_len, C.byref(actor.c(keep)), seed,
                                               out))
        return [GenSample(o.id, o.prompt_len, o.target_output_len, o.generated, o.kv_bytes) for o in out[:n]]

    def kv_bytes_per_token(self, spec: ModelSpec) -> float:
        keep: list = []
        v = C.c_double()
        check(self.lib, self.lib.fp_kv_bytes_per_token(C.byref(spec.c(keep)), C.byref(v)))
        return v.value

    # --- planner / simulation --------------------------------------------------------------
    def plan_migration(self, time: float, samples: list, r_t: int, cfg: GenSimConfig) -> MigrationPlan:
        keep: list = []
        arr = (_lib.Remaining * max(len(samples), 1))()
        for i, s in enumerate(samples):
            arr[i] = _lib.Remaining(s.id, s.instance, s.kv_bytes, s.generated, s.prompt_len, int(s.admitted))
        h = C.c_void_p()
        check(self.lib, self.lib.fp_plan_migration(time, arr, len(samples), r_t, C.byref(cfg.c(keep)), C.byref(h)))
        try:
            info = _lib.PlanInfo()
            check(self.lib, self.lib.fp_plan_info_get(h, C.byref(info), None, None))
            d = (C.c_int32 * max(info.n_destinations, 1))()
            m = (C.c_int32 * max(info.n_migrated, 1))()
            check(self.lib, self.lib.fp_plan_info_get(h, None, d, m))
            return _plan_from(info, d[:info.n_destinations], m[:info.n_migrated])
        finally:
            self.lib.fp_plan_free(h)

    def result_from_handle(self, h) -> GenStageResult:
        info = _lib.ResultInfo()
        check(self.lib, self.lib.fp_result_info_get(h, C.byref(info)))
        fin = (C.c_double * max(info.n_samples, 1))()
        ev = (_lib.Event * max(info.n_events, 1))()
        d = (C.c_int32 * max(info.plan.n_destinations, 1))()
        m = (C.c_int32 * max(info.plan.n_migrated, 1))()
        check(self.lib, self.lib.fp_result_arrays(h, fin, ev, d, m))
        n = C.c_size_t(0)
        check(self.lib, self.lib.fp_result_timeline(h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        check(self.lib, self.lib.fp_result_timeline(h, buf, n.value + 1, C.byref(n)))
        events = [(e.time, e.instance, _lib.EVENT_KINDS[e.kind], e.sample) for e in ev[:info.n_events]]
        return GenStageResult(info.gen_end, info.inf_end, info.total,
                              _plan_from(info.plan, d[:info.plan.n_destinations], m[:info.plan.n_migrated]),
                              bool(info.triggered), list(fin[:info.n_samples]), events, buf.value.decode())

    def _result(self, fn, *args) -> GenStageResult:
        h = C.c_void_p()
        check(self.lib, fn(*args, C.byref(h)))
        try:
            return self.result_from_handle(h)
        finally:
            self.lib.fp_result_free(h)

    def simulate_serial(self, batch: list, cfg: GenSimConfig) -> GenStageResult:
        keep: list = []
        return self._result(self.lib.fp_simulate_serial, batch_to_c(batch, keep), len(batch), C.byref(cfg.c(keep)))

    def simulate_fused(self, batch: list, cfg: GenSimConfig, r_t: int) -> GenStageResult:
        keep: list = []
        return self._result(self.lib.fp_simulate_fused, batch_to_c(batch, keep), len(batch), C.byref(cfg.c(keep)),
                            r_t)

    def sweep_threshold(self, batch: list, cfg: GenSimConfig, ratios: list | None = None) -> SweepResult:
        keep: list = []
        ratios = list(ratios or [])
        rr = (C.c_double * max(len(ratios), 1))(*ratios)
        cap = max(len(ratios), 19)
        curve = (_lib.SweepPoint * cap)()
        nc, best, serial = C.c_int32(), C.c_int32(), C.c_double()
        check(self.lib, self.lib.fp_sweep_threshold(batch_to_c(batch, keep), len(batch), C.byref(cfg.c(keep)), rr,
                                                    len(ratios), curve, C.byref(nc), C.byref(best),
                                                    C.byref(serial)))
        return SweepResult([(p.ratio, p.r_t, p.fused_total) for p in curve[:nc.value]], best.value, serial.value)

    def fused_trigger(self, batch: list, cfg: GenSimConfig, r_t: int) -> dict:
        """Product-library extension: trigger state, plan and moves the GPU executor takes."""
        keep: list = []
        b, c = batch_to_c(batch, keep), C.byref(cfg.c(keep))
        trig, ns, nm = C.c_int32(), C.c_int32(), C.c_int32()
        info = _lib.PlanInfo()
        check(self.lib, self.lib.fp_fused_trigger(b, len(batch), c, r_t, C.byref(trig), C.byref(info), None,
                                                  C.byref(ns), None, None, None, C.byref(nm)))
        st = (_lib.Remaining * max(ns.value, 1))()
        ms, mf, mt = ((C.c_int32 * max(nm.value, 1))() for _ in range(3))
        check(self.lib, self.lib.fp_fused_trigger(b, len(batch), c, r_t, C.byref(trig), C.byref(info), st,
                                                  C.byref(ns), ms, mf, mt, C.byref(nm)))
        return {"triggered": bool(trig.value), "time": info.trigger_time,
                "state": [Remaining(r.id, r.instance, r.kv_bytes, r.generated, r.prompt_len, bool(r.admitted))
                          for r in st[:ns.value]],
                "plan": _plan_from(info, [], []),
                "moves": list(zip(ms[:nm.value], mf[:nm.value], mt[:nm.value]))}

    # --- numerics --------------------------------------------------------------------------
    def _gae(self, fn, rewards, values, gamma, lam) -> np.ndarray:
        r = np.ascontiguousarray(rewards, dtype=np.float64)
        v = np.ascontiguousarray(values, dtype=np.float64)
        if len(r) < 1 or len(v) != len(r) + 1:  # the C ABI cannot see array lengths (numerics.cpp:12-14)
            raise _lib.ConfigError(_lib.FP_EINVAL, "GaeInputs: need T >= 1 rewards and T+1 values")
        out = np.zeros(max(len(r), 1), dtype=np.float64)
        dp = C.POINTER(C.c_double)
        check(self.lib, fn(r.ctypes.data_as(dp), v.ctypes.data_as(dp), len(r), gamma, lam, out.ctypes.data_as(dp)))
        return out[:len(r)]

    def balance_minibatch(self, lengths, dp: int) -> list:
        """balance_minibatch (workflow.hpp:63-66): sample indices per DP group."""
        n = len(lengths)
        ln = (C.c_int32 * max(n, 1))(*[int(x) for x in lengths])
        order = (C.c_int32 * max(n, 1))()
        off = (C.c_int32 * (max(dp, 0) + 1))()
        check(self.lib, self.lib.fp_balance_minibatch(ln, n, dp, None, order, off))
        return [list(order[off[g]:off[g + 1]]) for g in range(dp)]

    def gae_recursive(self, rewards, values, gamma=0.99, lam=0.95) -> np.ndarray:
        return self._gae(self.lib.fp_gae_recursive, rewards, values, gamma, lam)

    def gae_matrix(self, rewards, values, gamma=0.99, lam=0.95) -> np.ndarray:
        return self._gae(self.lib.fp_gae_matrix, rewards, values, gamma, lam)


def timeline_text(result: GenStageResult) -> str:
    return result.timeline
