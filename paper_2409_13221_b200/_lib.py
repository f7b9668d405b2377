"""ctypes view of the C ABIs (include/fp_sched.h, include/fp_engine.h).

`load()` opens the in-tree product library paper_2409_13221_b200/lib/
libfuseplan_b200.so and raises if it is missing — there is no Python or CPU
fallback for any product path. `load(path)` opens another library exporting
fp_sched.h (the oracle build of the reference sources, oracle/_ref/
libfuseplan_ref.so) for parity tests.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
PRODUCT_LIB = PKG / "lib" / "libfuseplan_b200.so"

FP_OK, FP_EINVAL, FP_EINFEASIBLE, FP_EINTERNAL = 0, 2, 3, 4
EVENT_KINDS = ["admit", "finish", "trigger", "migrate_out", "migrate_in", "join_inference", "gen_end", "inf_end"]


class FpError(RuntimeError):
    """Error returned across the C ABI; `.status` is the FP_* code."""

    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


class ConfigError(FpError):
    pass


class InfeasibleError(FpError):
    pass


class ModelSpec(C.Structure):
    _fields_ = [("name", C.c_char_p), ("num_layers", C.c_int32), ("num_heads", C.c_int32),
                ("hidden_size", C.c_int32), ("intermediate_size", C.c_int32)]


class CostModel(C.Structure):
    _fields_ = [("time_per_token_coeff", C.c_double), ("backward_forward_ratio", C.c_double),
                ("activation_bytes_coeff", C.c_double), ("decode_step_base", C.c_double),
                ("comm_bandwidth", C.c_double)]


class ClusterSpec(C.Structure):
    _fields_ = [("num_gpus", C.c_int32), ("gpus_per_node", C.c_int32),
                ("activation_capacity_per_stage", C.c_double), ("kv_capacity_per_instance", C.c_double),
                ("bs_max", C.c_int32), ("interconnect_bandwidth", C.c_double)]


class GenConfig(C.Structure):
    _fields_ = [("actor", ModelSpec), ("num_instances", C.c_int32), ("instance_gpus", C.c_int32),
                ("num_tasks", C.c_int32), ("tasks", C.POINTER(ModelSpec)), ("task_names", C.POINTER(C.c_char_p)),
                ("cluster", ClusterSpec), ("cost", CostModel)]


class GenSample(C.Structure):
    _fields_ = [("id", C.c_int32), ("prompt_len", C.c_int32), ("target_output_len", C.c_int32),
                ("generated", C.c_int32), ("kv_bytes", C.c_double)]


class LengthDist(C.Structure):
    _fields_ = [("kind", C.c_int32), ("median", C.c_double), ("p999_ratio", C.c_double), ("max_len", C.c_int32),
                ("empirical", C.POINTER(C.c_int32)), ("n_empirical", C.c_int32)]


class Remaining(C.Structure):
    _fields_ = [("id", C.c_int32), ("instance", C.c_int32), ("kv_bytes", C.c_double), ("generated", C.c_int32),
                ("prompt_len", C.c_int32), ("admitted", C.c_int32)]


class Event(C.Structure):
    _fields_ = [("time", C.c_double), ("instance", C.c_int32), ("kind", C.c_int32), ("sample", C.c_int32)]


class PlanInfo(C.Structure):
    _fields_ = [("trigger_time", C.c_double), ("r_t", C.c_int32), ("m", C.c_int32), ("mechanism", C.c_int32),
                ("no_op", C.c_int32), ("overhead", C.c_double), ("n_destinations", C.c_int32),
                ("n_migrated", C.c_int32)]


class ResultInfo(C.Structure):
    _fields_ = [("gen_end", C.c_double), ("inf_end", C.c_double), ("total", C.c_double), ("triggered", C.c_int32),
                ("n_samples", C.c_int32), ("n_events", C.c_int32), ("plan", PlanInfo)]


class SweepPoint(C.Structure):
    _fields_ = [("ratio", C.c_double), ("r_t", C.c_int32), ("fused_total", C.c_double)]


class ModelDims(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("hidden", C.c_int32), ("num_heads", C.c_int32),
                ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32), ("vocab", C.c_int32)]


class EngineSetup(C.Structure):
    _fields_ = [("actor", ModelDims), ("ref", ModelDims), ("critic", ModelDims), ("reward", ModelDims),
                ("weight_seed", C.c_uint64), ("max_prompt", C.c_int32), ("max_new", C.c_int32),
                ("max_samples", C.c_int32), ("max_live", C.c_int32), ("kv_pool_bytes", C.c_int64),
                ("max_prefill_tokens", C.c_int32), ("max_infer_tokens", C.c_int32), ("rope_theta", C.c_float),
                ("device", C.c_int32)]


class RunOptions(C.Structure):
    _fields_ = [("token_mode", C.c_int32), ("schedule", C.c_int32), ("temperature", C.c_float),
                ("token_seed", C.c_uint64), ("sample_seed", C.c_uint64), ("kl_beta", C.c_float),
                ("gamma", C.c_float), ("lam", C.c_float), ("claim_tokens", C.c_int32), ("run_ahead", C.c_int32),
                ("resident", C.c_int32), ("probe_attention", C.c_int32), ("handoff_dp", C.c_int32),
                ("claim_max_live", C.c_int32), ("eos_id", C.c_int32), ("eos_lag", C.c_int32),
                ("online_trigger", C.c_int32), ("top_k", C.c_int32), ("top_p", C.c_float)]


class Comm(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("shm_name", C.c_char_p)]


class ExecStats(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("gen_seconds", C.c_double), ("trigger_seconds", C.c_double),
                ("migrate_seconds", C.c_double), ("infer_busy_seconds", C.c_double),
                ("decode_gpu_seconds", C.c_double), ("decode_steps", C.c_int64), ("decode_rows", C.c_int64),
                ("decode_ctx_tokens", C.c_int64), ("prefill_tokens", C.c_int64), ("infer_tokens", C.c_int64),
                ("infer_samples", C.c_int64), ("migrated_in", C.c_int64), ("migrated_bytes", C.c_int64),
                ("total_resp", C.c_int64), ("gpu_launches", C.c_int64), ("attn_probe_ms", C.c_double),
                ("attn_probe_bytes", C.c_double), ("attn_probe_launches", C.c_int64), ("ipc_seconds", C.c_double),
                ("eos_retired", C.c_int64), ("overrun_rows", C.c_int64), ("online", C.c_int32)]


P = C.POINTER
_i32p, _i64p, _f32p, _f64p, _vp = P(C.c_int32), P(C.c_int64), P(C.c_float), P(C.c_double), C.c_void_p

SCHED_SYMBOLS = {
    "fp_last_error": (C.c_char_p, []),
    "fp_sample_lengths": (C.c_int, [P(LengthDist), C.c_int32, C.c_uint64, _i32p]),
    "fp_load_length_file": (C.c_int, [C.c_char_p, _i32p, C.c_int32, _i32p]),
    "fp_make_batch": (C.c_int, [P(LengthDist), C.c_int32, C.c_int32, P(ModelSpec), C.c_uint64, P(GenSample)]),
    "fp_kv_bytes_per_token": (C.c_int, [P(ModelSpec), _f64p]),
    "fp_plan_migration": (C.c_int, [C.c_double, P(Remaining), C.c_int32, C.c_int32, P(GenConfig), P(_vp)]),
    "fp_plan_info_get": (C.c_int, [_vp, P(PlanInfo), _i32p, _i32p]),
    "fp_plan_free": (None, [_vp]),
    "fp_simulate_serial": (C.c_int, [P(GenSample), C.c_int32, P(GenConfig), P(_vp)]),
    "fp_simulate_fused": (C.c_int, [P(GenSample), C.c_int32, P(GenConfig), C.c_int32, P(_vp)]),
    "fp_result_info_get": (C.c_int, [_vp, P(ResultInfo)]),
    "fp_result_arrays": (C.c_int, [_vp, _f64p, P(Event), _i32p, _i32p]),
    "fp_result_timeline": (C.c_int, [_vp, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "fp_result_free": (None, [_vp]),
    "fp_sweep_threshold": (C.c_int, [P(GenSample), C.c_int32, P(GenConfig), _f64p, C.c_int32, P(SweepPoint), _i32p,
                                     _i32p, _f64p]),
    "fp_balance_minibatch": (C.c_int, [_i32p, C.c_int32, C.c_int32, _i32p, _i32p, _i32p]),
    "fp_gae_recursive": (C.c_int, [_f64p, _f64p, C.c_int32, C.c_double, C.c_double, _f64p]),
    "fp_gae_matrix": (C.c_int, [_f64p, _f64p, C.c_int32, C.c_double, C.c_double, _f64p]),
}

ENGINE_SYMBOLS = {
    "fp_fused_trigger": (C.c_int, [P(GenSample), C.c_int32, P(GenConfig), C.c_int32, _i32p, P(PlanInfo),
                                   P(Remaining), _i32p, _i32p, _i32p, _i32p, _i32p]),
    "fp_engine_create": (C.c_int, [P(EngineSetup), P(_vp)]),
    "fp_engine_destroy": (None, [_vp]),
    "fp_engine_model_size": (C.c_int, [_vp, C.c_int32, _i64p, _i64p]),
    "fp_engine_broadcast_model": (C.c_int, [_vp, C.c_int32, C.c_int32, P(Comm), _f64p]),
    "fp_engine_model_ptr": (C.c_int, [_vp, C.c_int32, P(C.c_void_p), _i64p]),
    "fp_engine_reinit_model": (C.c_int, [_vp, C.c_int32, C.c_uint64]),
    "fp_engine_load_weights": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, _vp, C.c_int64]),
    "fp_engine_model_checksum": (C.c_int, [_vp, C.c_int32, P(C.c_uint64)]),
    "fp_engine_kv_bytes_per_token": (C.c_int, [_vp, _i64p]),
    "fp_synthetic_prompts": (C.c_int, [_vp, C.c_int32, C.c_uint64, _i32p]),
    "fp_execute": (C.c_int, [_vp, P(GenSample), C.c_int32, P(GenConfig), C.c_int32, P(RunOptions), P(Comm), _i32p,
                             P(_vp)]),
    "fp_exec_stats_get": (C.c_int, [_vp, P(ExecStats)]),
    "fp_exec_experience": (C.c_int, [_vp, _i64p, _i32p, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p, _f32p]),
    "fp_exec_finish": (C.c_int, [_vp, _f64p, _i32p]),
    "fp_exec_decision": (C.c_int, [_vp, P(_vp)]),
    "fp_exec_moves": (C.c_int, [_vp, _i32p, _i32p, _i32p, _i32p]),
    "fp_exec_received": (C.c_int, [_vp, _i32p, _i32p, _i32p]),
    "fp_exec_trigger_state": (C.c_int, [_vp, _f64p, _i32p, P(Remaining)]),
    "fp_exec_handoff": (C.c_int, [_vp, _i32p, _i32p, _i32p, _i32p, _i32p, _i64p, P(C.c_void_p), _f64p, _i64p,
                                  _i64p]),
    "fp_exec_handoff_download": (C.c_int, [_vp, P(C.c_void_p)]),
    "fp_exec_steps": (C.c_int, [_vp, _i32p, _i32p, _f32p, _i64p]),
    "fp_exec_free": (None, [_vp]),
    "fp_k_init_bf16": (C.c_int, [_vp, C.c_int64, C.c_uint64, C.c_uint64, C.c_float, _vp]),
    "fp_k_gemm_bf16": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, C.c_int32, _vp]),
    "fp_k_gemm_f32": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, C.c_int32, _vp]),
    "fp_k_gemm_f32_residual": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, _vp]),
    "fp_k_gemm_splits": (C.c_int, [C.c_int32, C.c_int32]),
    "fp_k_gemm_trace": (C.c_int, [_vp]),
    "fp_k_gemm_swiglu": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, _vp]),
    "fp_k_gemm_swiglu_decode": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, _vp]),
    "fp_k_qkv_rope": (C.c_int, [_vp, C.c_int32, _vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp, C.c_int32,
                                C.c_float, _vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, _vp, _vp]),
    "fp_k_vocab": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, C.c_int32, C.c_float, _vp, _vp, _vp,
                             C.c_uint64, _vp, _vp, _vp]),
    "fp_k_decode_chain": (C.c_int, [_vp] * 11 + [_vp, _vp, C.c_int32, C.c_int32, _vp, C.c_int32, _vp, _vp, C.c_int32,
                                   C.c_float] + [C.c_int32] * 6 + [_vp]),
    "fp_k_vocab_filtered": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int32, C.c_float, C.c_int32, C.c_float,
                                      _vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp]),
    "fp_k_add_norm": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp, C.c_int32, C.c_int32, _vp]),
    "fp_k_embed_norm": (C.c_int, [_vp, _vp, C.c_int32, _vp, C.c_int32, _vp, _vp, _vp, _vp]),
    "fp_k_rms_norm_rows": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, _vp]),
    "fp_k_attn_decode": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp, C.c_int32, C.c_int32,
                                   C.c_int32, _vp, C.c_int32, _vp, _vp, C.c_int32, _vp, _vp]),
    "fp_k_attn_trace": (None, [_vp]),
    "fp_k_attn_workspace_bytes": (C.c_int64, [C.c_int32] * 5),
    "fp_k_attn_items": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp]),
    "fp_k_attn_decode_ws": (C.c_int, [_vp, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _vp, C.c_int32, C.c_int32,
                                      C.c_int32, _vp, C.c_int32, _vp, _vp, _vp, C.c_int32, _vp, _vp, _vp]),
    "fp_k_attn_varlen": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int32, _i32p, _vp, C.c_int32, _vp,
                                   _vp]),
    "fp_k_attn_prefill_trace": (C.c_int, [_vp]),
    "fp_k_set_packed_persistent": (C.c_int, [C.c_int]),
    "fp_k_set_pair_gemm": (C.c_int, [C.c_int]),
    "fp_k_set_attn_cut": (C.c_int, [C.c_int]),
    "fp_k_attn_varlen_mma": (C.c_int, [_vp, _vp, _vp, C.c_int32, C.c_int32, C.c_int32, _i32p, _vp, C.c_int32,
                                       _vp, _vp]),
    "fp_k_postprocess": (C.c_int, [C.c_int32, _vp, _vp, _vp, _vp, _vp, C.c_float, C.c_float, C.c_float, _vp, _vp,
                                   _vp, _vp, _vp]),
}

_cache: dict[str, C.CDLL] = {}


def load(path: str | os.PathLike | None = None, engine: bool | None = None) -> C.CDLL:
    """Open a library exporting fp_sched.h (and fp_engine.h for the product)."""
    p = Path(path) if path is not None else PRODUCT_LIB
    key = str(p.resolve()) if p.exists() else str(p)
    if key in _cache:
        return _cache[key]
    if not p.exists():
        raise FileNotFoundError(
            f"native library not built: {p} (run `python -c 'import __graft_entry__ as g; g.build()'`); "
            "there is no fallback path")
    lib = C.CDLL(str(p), mode=C.RTLD_LOCAL)
    symbols = dict(SCHED_SYMBOLS)
    if engine is None:
        engine = path is None
    if engine:
        symbols.update(ENGINE_SYMBOLS)
    for name, (res, args) in symbols.items():
        fn = getattr(lib, name)  # AttributeError: symbol missing from the ABI
        fn.restype = res
        fn.argtypes = args
    _cache[key] = lib
    return lib


def check(lib: C.CDLL, status: int) -> None:
    if status == FP_OK:
        return
    msg = (lib.fp_last_error() or b"").decode(errors="replace")
    if status == FP_EINVAL:
        raise ConfigError(status, msg)
    if status == FP_EINFEASIBLE:
        raise InfeasibleError(status, msg)
    raise FpError(status, msg)
