"""Python host mirror of the engine C ABI (include/fp_engine.h).

`Engine(workload)` creates one B200 engine (weights of the four models, paged
KV pool, workspaces) on a device; `Engine.execute(...)` runs the gen+inf stage
(serial = stage barrier, or fused) for a batch, returning the experience
batch, measured statistics and the decision-clock result — the GPU
counterpart of Sched.simulate_serial / simulate_fused (genfuse.hpp:113-121).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check
from .configs import Dims, Workload
from .sched import GenSimConfig, Sched, batch_to_c

TOKEN_MODES = {"forced": 0, "greedy": 1, "sample": 2}
SCHEDULES = {"stage_barrier": 0, "serial": 0, "fused": 1}


def _dims(d: Dims) -> _lib.ModelDims:
    return _lib.ModelDims(d.num_layers, d.hidden, d.num_heads, d.num_kv_heads, d.head_dim, d.ffn, d.vocab)


@dataclass
class Experience:
    resp_off: np.ndarray
    tokens: np.ndarray
    logp_actor: np.ndarray
    logp_ref: np.ndarray
    values: np.ndarray
    kl: np.ndarray
    reward: np.ndarray
    adv: np.ndarray
    ret: np.ndarray
    score: np.ndarray

    def sample(self, i: int) -> dict:
        b, e = int(self.resp_off[i]), int(self.resp_off[i + 1])
        return {k: getattr(self, k)[b:e] for k in ("tokens", "logp_actor", "logp_ref", "values", "kl", "reward",
                                                   "adv", "ret")} | {"score": float(self.score[i])}


@dataclass
class ExecOutput:
    stats: dict
    experience: Experience
    finish_seconds: np.ndarray
    finish_instance: np.ndarray
    decision: object  # sched.GenStageResult
    moves: list       # (sample, from, to) in application order
    step_rows: np.ndarray = None  # per decode step of this rank: batch rows
    step_ms: np.ndarray = None    # per decode step: GPU ms
    handoff: dict = None          # handoff_dp > 0: order, group_off, packed_off, this rank's packed arrays
    received: list = None         # (sample, source rank) this rank pulled in at the migration
    trigger_state: tuple = None   # (time, [Remaining...]) the executed plan was taken on
    online: bool = False          # the trigger was taken online
    step_ctx: np.ndarray = None   # per decode step: visible context tokens summed over its rows


class Engine:
    def __init__(self, w: Workload, *, device: int = 0, weight_seed: int = 1234, max_samples: int | None = None,
                 max_live: int | None = None, kv_pool_bytes: int = 0, max_prefill_tokens: int = 16384,
                 max_infer_tokens: int = 16384, rope_theta: float = 10000.0):
        self.lib = _lib.load()
        self.workload = w
        n = max_samples or w.n_prompts
        setup = _lib.EngineSetup(_dims(w.actor), _dims(w.ref), _dims(w.critic), _dims(w.reward), weight_seed,
                                 w.prompt_len, w.max_new, n, max_live or n, kv_pool_bytes, max_prefill_tokens,
                                 max_infer_tokens, rope_theta, device)
        self.setup = setup
        h = C.c_void_p()
        check(self.lib, self.lib.fp_engine_create(C.byref(setup), C.byref(h)))
        self.h = h
        self.sched = Sched(self.lib)

    def close(self):
        if getattr(self, "h", None):
            self.lib.fp_engine_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def model_size(self, m: int) -> tuple:
        b, p = C.c_int64(), C.c_int64()
        check(self.lib, self.lib.fp_engine_model_size(self.h, m, C.byref(b), C.byref(p)))
        return b.value, p.value

    def kv_bytes_per_token(self) -> int:
        v = C.c_int64()
        check(self.lib, self.lib.fp_engine_kv_bytes_per_token(self.h, C.byref(v)))
        return v.value

    def _handoff(self, x, n: int) -> dict:
        dp, gb, ge = C.c_int32(), C.c_int32(), C.c_int32()
        check(self.lib, self.lib.fp_exec_handoff(x, C.byref(dp), None, None, None, None, None, None, None, None,
                                                 None))
        order = np.zeros(n, dtype=np.int32)
        goff = np.zeros(dp.value + 1, dtype=np.int32)
        poff = np.zeros(n + 1, dtype=np.int64)
        sec, nb, pb = C.c_double(), C.c_int64(), C.c_int64()
        i32 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int32))  # noqa: E731
        check(self.lib, self.lib.fp_exec_handoff(x, C.byref(dp), C.byref(gb), C.byref(ge), i32(order), i32(goff),
                                                 poff.ctypes.data_as(C.POINTER(C.c_int64)), None, C.byref(sec),
                                                 C.byref(nb), C.byref(pb)))
        k0, k1 = goff[gb.value], goff[ge.value]
        T = int(poff[k1] - poff[k0])
        arrays = [np.zeros(max(T, 1), dtype=np.int32)] + [np.zeros(max(T, 1), dtype=np.float32) for _ in range(7)]
        score = np.zeros(max(k1 - k0, 1), dtype=np.float32)
        host = (C.c_void_p * 9)(*[a.ctypes.data for a in arrays], score.ctypes.data)
        check(self.lib, self.lib.fp_exec_handoff_download(x, host))
        names = ("tokens", "logp_actor", "logp_ref", "values", "kl", "reward", "adv", "ret")
        out = {"dp": dp.value, "order": order, "group_off": goff, "packed_off": poff, "group_begin": gb.value,
               "group_end": ge.value, "seconds": sec.value, "bytes": nb.value, "peer_bytes": pb.value,
               "score": score[:k1 - k0]}
        out.update({k: a[:T] for k, a in zip(names, arrays)})
        return out

    MODELS = {"actor": 0, "ref": 1, "critic": 2, "reward": 3}
    TENSORS = {"embed": 0, "wqkv": 1, "wo": 2, "wg": 3, "wu": 4, "wd": 5, "ln1": 6, "ln2": 7, "lnf": 8, "head": 9,
               "vhead": 10}

    def load_weights(self, model: str, tensors: dict) -> None:
        """fp_engine_load_weights for every tensor of `tensors` (model_oracle.make_weights layout:
        embed, layers[l][wqkv|wo|wg|wu|wd|ln1|ln2], lnf, head | vhead). Matrices are converted to
        bf16 (round to nearest even), norm gains stay fp32."""
        m = self.MODELS[model]

        def put(name, layer, a):
            a = np.ascontiguousarray(a, dtype=np.float32)
            if name in ("ln1", "ln2", "lnf"):
                buf = a
            else:  # fp32 -> bf16 bits, round to nearest even
                b = a.view(np.uint32).astype(np.uint64)
                buf = ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)
            check(self.lib, self.lib.fp_engine_load_weights(self.h, m, self.TENSORS[name], layer,
                                                            buf.ctypes.data_as(C.c_void_p), buf.size))

        for name in ("embed", "lnf", "head", "vhead"):
            if name in tensors:
                put(name, 0, tensors[name])
        for l, lw in enumerate(tensors.get("layers", [])):
            for name, a in lw.items():
                put(name, l, a)

    def broadcast_model(self, model: str, src: int, rank: int, world: int, shm_name: str | None) -> float:
        """Weight sync over NVLink (fp_engine_broadcast_model): every rank calls it; returns seconds."""
        comm = _lib.Comm(rank, world, shm_name.encode() if shm_name else None)
        t = C.c_double()
        check(self.lib, self.lib.fp_engine_broadcast_model(self.h, self.MODELS[model], src, C.byref(comm),
                                                           C.byref(t)))
        return t.value

    def reinit_model(self, model: str, seed: int) -> None:
        check(self.lib, self.lib.fp_engine_reinit_model(self.h, self.MODELS[model], seed))

    def model_checksum(self, model: str) -> int:
        v = C.c_uint64()
        check(self.lib, self.lib.fp_engine_model_checksum(self.h, self.MODELS[model], C.byref(v)))
        return v.value

    def synthetic_prompts(self, n: int, token_seed: int) -> np.ndarray:
        out = np.zeros((n, self.setup.max_prompt), dtype=np.int32)
        check(self.lib, self.lib.fp_synthetic_prompts(self.h, n, token_seed,
                                                      out.ctypes.data_as(C.POINTER(C.c_int32))))
        return out

    def execute(self, batch: list, cfg: GenSimConfig, r_t: int = 0, *, token_mode: str = "forced",
                schedule: str = "fused", temperature: float = 1.0, token_seed: int = 7, sample_seed: int = 11,
                kl_beta: float = 0.05, gamma: float = 1.0, lam: float = 0.95, claim_tokens: int = 8192,
                run_ahead: int = 4, rank: int = 0, world: int = 1, shm_name: str | None = None,
                prompts: np.ndarray | None = None, resident: bool = False,
                probe_attention: bool = False, handoff_dp: int = 0, claim_max_live: int = 0, eos_id: int = -1,
                eos_lag: int = 1, online_trigger: bool = False, top_k: int = 0, top_p: float = 1.0) -> ExecOutput:
        keep: list = []
        n = len(batch)
        opts = _lib.RunOptions(TOKEN_MODES[token_mode], SCHEDULES[schedule], temperature, token_seed, sample_seed,
                               kl_beta, gamma, lam, claim_tokens, run_ahead, int(resident), int(probe_attention),
                               handoff_dp, claim_max_live, eos_id, eos_lag, int(online_trigger), top_k, top_p)
        comm = _lib.Comm(rank, world, shm_name.encode() if shm_name else None)
        pp = None
        if prompts is not None:
            prompts = np.ascontiguousarray(prompts, dtype=np.int32)
            pp = prompts.ctypes.data_as(C.POINTER(C.c_int32))
        x = C.c_void_p()
        check(self.lib, self.lib.fp_execute(self.h, batch_to_c(batch, keep), n, C.byref(cfg.c(keep)), r_t,
                                            C.byref(opts), C.byref(comm), pp, C.byref(x)))
        try:
            st = _lib.ExecStats()
            check(self.lib, self.lib.fp_exec_stats_get(x, C.byref(st)))
            stats = {k: getattr(st, k) for k, _ in _lib.ExecStats._fields_}
            T = st.total_resp
            f32 = lambda: np.zeros(max(T, 1), dtype=np.float32)  # noqa: E731
            arrs = {k: f32() for k in ("logp_actor", "logp_ref", "values", "kl", "reward", "adv", "ret")}
            tokens = np.zeros(max(T, 1), dtype=np.int32)
            off = np.zeros(n + 1, dtype=np.int64)
            score = np.zeros(n, dtype=np.float32)
            fp = lambda a: a.ctypes.data_as(C.POINTER(C.c_float))  # noqa: E731
            check(self.lib, self.lib.fp_exec_experience(
                x, off.ctypes.data_as(C.POINTER(C.c_int64)), tokens.ctypes.data_as(C.POINTER(C.c_int32)),
                fp(arrs["logp_actor"]), fp(arrs["logp_ref"]), fp(arrs["values"]), fp(arrs["kl"]),
                fp(arrs["reward"]), fp(arrs["adv"]), fp(arrs["ret"]), fp(score)))
            exp = Experience(off, tokens[:T], *(arrs[k][:T] for k in ("logp_actor", "logp_ref", "values", "kl",
                                                                        "reward", "adv", "ret")), score)
            fin = np.zeros(n, dtype=np.float64)
            inst = np.zeros(n, dtype=np.int32)
            check(self.lib, self.lib.fp_exec_finish(x, fin.ctypes.data_as(C.POINTER(C.c_double)),
                                                    inst.ctypes.data_as(C.POINTER(C.c_int32))))
            hres = C.c_void_p()
            check(self.lib, self.lib.fp_exec_decision(x, C.byref(hres)))
            try:
                decision = self.sched.result_from_handle(hres)
            finally:
                self.lib.fp_result_free(hres)
            nm = C.c_int32()
            check(self.lib, self.lib.fp_exec_moves(x, C.byref(nm), None, None, None))
            ms, mf, mt = ((C.c_int32 * max(nm.value, 1))() for _ in range(3))
            check(self.lib, self.lib.fp_exec_moves(x, C.byref(nm), ms, mf, mt))
            moves = list(zip(ms[:nm.value], mf[:nm.value], mt[:nm.value]))
            ns = C.c_int32()
            check(self.lib, self.lib.fp_exec_steps(x, C.byref(ns), None, None, None))
            srows = np.zeros(max(ns.value, 1), dtype=np.int32)
            sms = np.zeros(max(ns.value, 1), dtype=np.float32)
            sctx = np.zeros(max(ns.value, 1), dtype=np.int64)
            check(self.lib, self.lib.fp_exec_steps(x, C.byref(ns), srows.ctypes.data_as(C.POINTER(C.c_int32)),
                                                   sms.ctypes.data_as(C.POINTER(C.c_float)),
                                                   sctx.ctypes.data_as(C.POINTER(C.c_int64))))
            handoff = self._handoff(x, n) if handoff_dp > 0 else None
            nr = C.c_int32()
            check(self.lib, self.lib.fp_exec_received(x, C.byref(nr), None, None))
            rs, rf = ((C.c_int32 * max(nr.value, 1))() for _ in range(2))
            check(self.lib, self.lib.fp_exec_received(x, C.byref(nr), rs, rf))
            tt, nt = C.c_double(), C.c_int32()
            check(self.lib, self.lib.fp_exec_trigger_state(x, C.byref(tt), C.byref(nt), None))
            tst = (_lib.Remaining * max(nt.value, 1))()
            check(self.lib, self.lib.fp_exec_trigger_state(x, C.byref(tt), C.byref(nt), tst))
            state = (tt.value, [(r.id, r.instance, r.kv_bytes, r.generated, r.prompt_len, bool(r.admitted))
                                for r in tst[:nt.value]])
            return ExecOutput(stats, exp, fin, inst, decision, moves, srows[:ns.value], sms[:ns.value], handoff,
                              list(zip(rs[:nr.value], rf[:nr.value])), state, bool(st.online), sctx[:ns.value])
        finally:
            self.lib.fp_exec_free(x)
