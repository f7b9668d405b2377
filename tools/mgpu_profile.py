"""Per-rank phase times of the fused schedule on G GPUs (torchrun, one rank per GPU).

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/mgpu_profile.py [reps]
"""
import json
import os
import sys
import time
import uuid

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
sched = sys.argv[2] if len(sys.argv) > 2 else "fused"
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dist.init_process_group("gloo")
torch.cuda.set_device(local)
w = scaled(WORKLOADS["gpt2s"], n_prompts=512 * world)
eng = Engine(w, device=local, max_samples=w.n_prompts, max_live=min(w.n_prompts, 2 * w.n_prompts // world))
batch = batch_for(w, eng.sched)
cfg = gen_config(w, world, calibrated=True)
r_t = round((float(sys.argv[3]) if len(sys.argv) > 3 else 0.2) * len(batch))
name = [f"/fp_prof_{uuid.uuid4().hex[:10]}" if rank == 0 else None]
dist.broadcast_object_list(name, src=0)
prompts = eng.synthetic_prompts(len(batch), 7)
for k in range(reps):
    dist.barrier()
    t0 = time.perf_counter()
    out = eng.execute(batch, cfg, r_t, token_mode="sample", schedule=sched, rank=rank, world=world,
                      shm_name=f"{name[0]}_{k}", prompts=prompts, resident=True)
    t1 = time.perf_counter()
    st = out.stats
    keys = ("wall_seconds", "gen_seconds", "trigger_seconds", "migrate_seconds", "ipc_seconds",
            "infer_busy_seconds", "decode_gpu_seconds", "decode_steps", "decode_rows", "infer_samples",
            "migrated_in", "migrated_bytes")
    row = {"rep": k, "rank": rank, "host_s": round(t1 - t0, 4)} | {x: (round(st[x], 4) if isinstance(st[x], float)
                                                                    else st[x]) for x in keys}
    rows = [None] * world
    dist.all_gather_object(rows, row)
    if rank == 0:
        for r in rows:
            print(json.dumps(r), flush=True)
eng.close()
dist.destroy_process_group()
