"""Worker for the multi-GPU tests (launched by torchrun, one rank per GPU).

Runs the toy workload on G ranks with the fused schedule (one-shot long-tail
migration at r_t) and, on rank 0, compares the gathered experience with a
single-GPU stage-barrier run of the same batch on the same device: per-row
kernels are batch-independent, so the two must agree bit for bit. Also checks
that the executed moves are the decision clock's (simulate_fused), and writes
a JSON summary to the path given as argv[1].
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


def main():
    out_path = sys.argv[1]
    mode = sys.argv[2] if len(sys.argv) > 2 else "forced"
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    w = scaled(WORKLOADS["toy"], n_prompts=64 * world, max_new=256, prompt_len=24)
    eng = Engine(w, device=local, max_samples=w.n_prompts, max_live=w.n_prompts)
    batch = batch_for(w, eng.sched)
    # KV-capped decision clock so that admission waves, the trigger and the
    # migration plan are non-trivial.
    kv_max = max(b.kv_bytes for b in batch)
    mech = sys.argv[3] if len(sys.argv) > 3 else "kv"
    cfg = gen_config(w, world, bs_max=64, kv_capacity=48 * kv_max, decode_step_base=1e-3,
                     interconnect_bandwidth=770e9 if mech == "kv" else 1e3)
    r_t = round(0.25 * len(batch))
    name = [f"/fp_test_{uuid.uuid4().hex[:10]}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    res = {}
    for rep in range(2):
        out = eng.execute(batch, cfg, r_t, token_mode=mode, schedule="fused", claim_tokens=2048, rank=rank,
                          world=world, shm_name=name[0] + f"_{rep}", handoff_dp=2 * world if rep else 0)
    h = out.handoff
    np.savez(f"{out_path}.rank{rank}.npz", **{k: np.asarray(v) for k, v in h.items()})
    res["stats"] = out.stats
    res["moves"] = out.moves
    ref_moves = None
    if rank == 0:
        fused = eng.sched.simulate_fused(batch, cfg, r_t)
        ref_moves = [(e[3], e[1]) for e in fused.events if e[2] == "migrate_in"]
        res["plan"] = {"mechanism": fused.plan.mechanism, "m": fused.plan.m, "destinations": fused.plan.destinations, "no_op": fused.plan.no_op,
                       "n_migrated": len(fused.plan.migrated), "trigger": fused.plan.trigger_time}
        res["moves_match"] = sorted((s, t) for s, _, t in out.moves) == sorted(ref_moves)
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
        # single-GPU stage-barrier run of the same batch on this device
        eng1 = Engine(w, device=local, max_samples=w.n_prompts, max_live=w.n_prompts)
        one = eng1.execute(batch, gen_config(w, 1, bs_max=64, kv_capacity=48 * kv_max), 0, token_mode=mode,
                           schedule="stage_barrier")
        a, b = out.experience, one.experience
        diffs = {k: int(np.sum(getattr(a, k) != getattr(b, k))) for k in
                 ("tokens", "logp_actor", "logp_ref", "values", "kl", "reward", "adv", "ret", "score")}
        res["diffs_vs_1gpu"] = diffs
        res["identical"] = all(v == 0 for v in diffs.values())
        res["max_abs"] = {k: float(np.max(np.abs(getattr(a, k).astype(np.float64) - getattr(b, k))))
                          for k in ("logp_actor", "logp_ref", "values", "adv", "ret")}
        res["n"] = len(batch)
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
        eng1.close()
        Path(out_path).write_text(json.dumps(res, default=lambda o: o if not hasattr(o, "__dict__") else o.__dict__))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
