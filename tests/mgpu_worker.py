"""Worker for the multi-rank tests (launched by torchrun, one rank per process).

Ranks normally own one GPU each; with FP_MGPU_SAME_DEVICE=1 every rank runs
its engine on cuda:0 (CUDA IPC works between processes on one device), so the
multi-rank executor — migration, cross-rank scoring queue, hand-off, weight
broadcast — runs on a 1-GPU box too.

Scenarios (argv[2]):
  clock-forced-kv | clock-greedy-kv | clock-forced-recompute
      fused schedule with the decision clock's trigger (bit-exact with
      simulate_fused): the samples the executor actually pulled in, gathered
      over ranks, must be simulate_fused's migrate_in events; experience
      bit-identical to a 1-GPU stage-barrier run (recompute: tokens exact).
  online-forced
      teacher-forced lengths, online trigger: the executed plan must equal
      plan_migration (reference library when built) on the published trigger
      state, fewer than r_t samples unfinished at the trigger, moves = what
      was pulled in, experience bit-identical to 1 GPU.
  online-eos
      free-run greedy generation retiring on an emitted EOS id (chosen as a
      token the model emits often), online trigger: experience and response
      lengths bit-identical to a 1-GPU free-run, every response ends at its
      first EOS or at max_new.
Writes a JSON summary to argv[1] (rank 0).
"""
import json
import os
import sys
import uuid
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402
from paper_2409_13221_b200.sched import Sched  # noqa: E402

KEYS = ("tokens", "logp_actor", "logp_ref", "values", "kl", "reward", "adv", "ret", "score")


def diffs(a, b):
    if len(a.resp_off) != len(b.resp_off) or not np.array_equal(a.resp_off, b.resp_off):
        return {"resp_off": -1}
    return {k: int(np.sum(getattr(a, k) != getattr(b, k))) for k in KEYS}


def main():
    out_path, scenario = sys.argv[1], sys.argv[2]
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    same = os.environ.get("FP_MGPU_SAME_DEVICE") == "1"
    local = 0 if same else int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    max_new = 256 if scenario.startswith("clock") else 192
    w = scaled(WORKLOADS["toy"], n_prompts=48 * world, max_new=max_new, prompt_len=24)
    eng = Engine(w, device=local, max_samples=w.n_prompts, max_live=w.n_prompts)
    batch = batch_for(w, eng.sched)
    # KV-capped decision clock so that admission waves, the trigger and the
    # migration plan are non-trivial
    kv_max = max(b.kv_bytes for b in batch)
    mech = "recompute" if scenario.endswith("recompute") else "kv"
    cfg = gen_config(w, world, bs_max=32, kv_capacity=36 * kv_max, decode_step_base=1e-3,
                     interconnect_bandwidth=770e9 if mech == "kv" else 1e3)
    cfg1 = gen_config(w, 1, bs_max=32, kv_capacity=36 * kv_max, decode_step_base=1e-3)
    r_t = round(0.3 * len(batch))
    name = [f"/fp_test_{uuid.uuid4().hex[:10]}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    kw = dict(schedule="fused", claim_tokens=1024, rank=rank, world=world)
    res = {"scenario": scenario, "same_device": same, "n": len(batch), "r_t": r_t}
    if scenario.startswith("clock"):
        mode = "greedy" if "greedy" in scenario else "forced"
        kw["token_mode"] = mode
        one_kw = dict(token_mode=mode)
    elif scenario == "online-forced":
        kw.update(token_mode="forced", online_trigger=True)
        one_kw = dict(token_mode="forced")
    elif scenario == "online-eos":
        # EOS = the most frequent emitted token of a short greedy run (rank 0, alone)
        eos = [None]
        if rank == 0:
            probe = eng.execute(batch[:16], gen_config(w, 1), 0, token_mode="greedy", schedule="stage_barrier")
            vals, cnt = np.unique(probe.experience.tokens, return_counts=True)
            eos[0] = int(vals[np.argmax(cnt)])
        dist.broadcast_object_list(eos, src=0)
        res["eos_id"] = eos[0]
        kw.update(token_mode="greedy", eos_id=eos[0], eos_lag=2)
        one_kw = dict(token_mode="greedy", eos_id=eos[0], eos_lag=0)
        # free-run reservations are prompt + max_new: cap the pool in those units
        kv_tok = eng.sched.kv_bytes_per_token(cfg.actor)
        cfg.cluster.kv_capacity_per_instance = 36 * (w.prompt_len + w.max_new) * kv_tok
        cfg1.cluster.kv_capacity_per_instance = cfg.cluster.kv_capacity_per_instance
    else:
        raise SystemExit(f"unknown scenario {scenario}")

    for rep in range(2):  # the second run exercises cached IPC mappings and the hand-off
        out = eng.execute(batch, cfg, r_t, shm_name=name[0] + f"_{rep}", handoff_dp=2 * world if rep else 0, **kw)
    np.savez(f"{out_path}.rank{rank}.npz", **{k: np.asarray(v) for k, v in out.handoff.items()})
    got = [None] * world
    dist.all_gather_object(got, {"received": out.received, "stats": out.stats, "moves": out.moves,
                                 "online": out.online, "state": out.trigger_state})
    res["stats"] = [g["stats"] for g in got]
    received = sorted((s, f, r) for r, g in enumerate(got) for s, f in g["received"])
    res["received"] = received
    if rank == 0:
        res["online"] = out.online
        res["moves"] = [list(m) for m in out.moves]
        res["moves_equal_received"] = sorted(tuple(m) for m in out.moves) == received
        if scenario.startswith("clock"):
            fused = eng.sched.simulate_fused(batch, cfg, r_t)
            res["plan"] = {"mechanism": fused.plan.mechanism, "m": fused.plan.m, "no_op": fused.plan.no_op,
                           "destinations": list(fused.plan.destinations), "n_migrated": len(fused.plan.migrated)}
            ref_in = sorted((e[3], e[1]) for e in fused.events if e[2] == "migrate_in")
            res["received_match_clock"] = sorted((s, r) for s, _, r in received) == ref_in
        else:
            t, state = out.trigger_state
            ref = ROOT / "oracle" / "_ref" / "libfuseplan_ref.so"
            sref = Sched(str(ref)) if ref.exists() else eng.sched
            res["plan_lib"] = "reference" if ref.exists() else "product"
            from paper_2409_13221_b200.sched import Remaining
            rem = [Remaining(*s) for s in state]
            plan = sref.plan_migration(t, rem, r_t, cfg)
            res["n_unfinished_at_trigger"] = len(state)
            res["plan"] = {"mechanism": plan.mechanism, "m": plan.m, "no_op": plan.no_op,
                           "destinations": list(plan.destinations), "n_migrated": len(plan.migrated)}
            # every executed move is a migrant of the reference plan, sent to one
            # of its destinations; the queued migrants all move
            queued = {s[0] for s in state if not s[5]} & set(plan.migrated)
            moved = {m[0] for m in out.moves}
            res["moves_within_plan"] = ((not plan.no_op or not out.moves) and moved <= set(plan.migrated)
                                        and all(m[2] in plan.destinations for m in out.moves) and queued <= moved)
    dist.barrier()
    # weight sync: rank 0 gets new actor weights, every rank pulls them
    c0 = eng.model_checksum("actor")
    if rank == 0:
        eng.reinit_model("actor", 4321)
    dist.barrier()
    t_bc = eng.broadcast_model("actor", 0, rank, world, name[0] + "_bc")
    sums = [None] * world
    dist.all_gather_object(sums, (c0, eng.model_checksum("actor"), t_bc))
    res["bcast"] = {"same": len({s[1] for s in sums}) == 1, "changed": all(s[1] != s[0] for s in sums),
                    "seconds": max(s[2] for s in sums)}
    if rank == 0:
        eng.reinit_model("actor", 1234)  # restore for the single-rank comparison
        one = eng.execute(batch, cfg1, 0, schedule="stage_barrier", **one_kw)
        a, b = out.experience, one.experience
        d = diffs(a, b)
        res["diffs_vs_1gpu"] = d
        res["identical"] = all(v == 0 for v in d.values())
        if d.get("resp_off") != -1:
            res["max_abs"] = {k: float(np.max(np.abs(getattr(a, k).astype(np.float64) - getattr(b, k))))
                              for k in ("logp_actor", "logp_ref", "values", "adv", "ret")}
        if scenario == "online-eos":
            eos = res["eos_id"]
            lens = np.diff(a.resp_off)
            ok = True
            for i in range(len(batch)):
                tk = a.tokens[a.resp_off[i]:a.resp_off[i + 1]]
                first = np.flatnonzero(tk == eos)
                ok &= (len(first) == 0 and len(tk) == w.max_new) or (len(first) > 0 and first[0] == len(tk) - 1)
            res["eos_semantics_ok"] = bool(ok)
            res["lengths"] = {"min": int(lens.min()), "max": int(lens.max()), "mean": float(lens.mean()),
                              "at_max_new": int(np.sum(lens == w.max_new))}
        # hand-off: every rank's packed DP groups == the gathered experience in
        # balance_minibatch order (pulled over NVLink from the scoring ranks)
        x = out.experience
        ho_ok, peer = True, 0
        for r in range(world):
            hr = np.load(f"{out_path}.rank{r}.npz")
            k0, k1 = hr["group_off"][int(hr["group_begin"])], hr["group_off"][int(hr["group_end"])]
            ids = hr["order"][k0:k1]
            idx = np.concatenate([np.arange(x.resp_off[s], x.resp_off[s + 1]) for s in ids])
            for k in ("tokens", "logp_actor", "logp_ref", "values", "kl", "reward", "adv", "ret"):
                ho_ok &= bool(np.array_equal(hr[k], getattr(x, k)[idx]))
            ho_ok &= bool(np.array_equal(hr["score"], x.score[ids]))
            peer += int(hr["peer_bytes"])
        res["handoff_ok"] = ho_ok
        res["handoff_peer_bytes"] = peer
        Path(out_path).write_text(json.dumps(res, default=lambda o: o if not hasattr(o, "__dict__") else o.__dict__))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
