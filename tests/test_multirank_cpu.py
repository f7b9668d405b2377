"""N > 1 host-side logic on CPU (gloo, world size 2 — no GPU needed).

Every rank computes the decision clock independently (that is how the GPU
executor works: no decision is communicated, only data). Here two gloo ranks
each compute the fused trigger / plan / moves and the round-robin shard for
the same batch; all-gathered results must agree bit for bit, shards must
partition the batch, and the moves must be exactly the migrate_out/migrate_in
pairs of the decision-clock timeline (simulate_fused).
"""
import os
import pickle
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled
    from paper_2409_13221_b200.sched import Sched
    s = Sched()
    w = scaled(WORKLOADS["1.3b"], n_prompts=256)
    batch = batch_for(w, s)
    kv_max = max(b.kv_bytes for b in batch)
    out = {}
    for G in (2, 4, 8):
        cfg = gen_config(w, G, bs_max=64, kv_capacity=48 * kv_max)
        for ratio in (0.1, 0.25):
            r_t = round(ratio * len(batch))
            t = s.fused_trigger(batch, cfg, r_t)
            f = s.simulate_fused(batch, cfg, r_t)
            outs = {e[3]: e[1] for e in f.events if e[2] == "migrate_out"}
            ins = {e[3]: e[1] for e in f.events if e[2] == "migrate_in"}
            consistent = sorted((sid, outs[sid], ins[sid]) for sid in ins) == sorted(t["moves"])
            mine = [i for i in range(len(batch)) if i % G == rank]
            out[(G, r_t)] = (t["time"], t["plan"].m, [(m.id, m.instance, m.generated, m.admitted) for m in t["state"]],
                             t["moves"], consistent, mine, f.plan.destinations)
    gathered = [None] * world
    dist.all_gather_object(gathered, pickle.dumps(out))
    if rank == 0:
        q.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def test_ranks_agree_on_decisions_and_shards():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    per_rank = [pickle.loads(g) for g in gathered]
    for key in per_rank[0]:
        a, b = per_rank[0][key], per_rank[1][key]
        assert a[:5] == b[:5], key          # identical decisions on both ranks
        assert a[4], key                    # moves == decision-clock timeline pairs
        G = key[0]
        # rank shards: round robin s % G; two ranks see disjoint shards
        assert set(a[5]).isdisjoint(b[5]) and all(s % G == 0 for s in a[5]) and all(s % G == 1 for s in b[5])
        # every move goes to one of the plan's destinations
        assert all(t in a[6] for _, _, t in a[3])
