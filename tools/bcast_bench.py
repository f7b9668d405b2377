"""Actor weight sync over NVLink (fp_engine_broadcast_model) on G GPUs.

    python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 tools/bcast_bench.py [workload]
"""
import os
import sys
import uuid

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
from paper_2409_13221_b200.configs import WORKLOADS, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
dist.init_process_group("gloo")
torch.cuda.set_device(local)
w = scaled(WORKLOADS[wl], n_prompts=8)
eng = Engine(w, device=local, max_samples=8, max_live=8)
import ctypes as C  # noqa: E402
nb = C.c_int64()
eng.lib.fp_engine_model_size(eng.h, 0, C.byref(nb), None)
name = [f"/fp_bc_{uuid.uuid4().hex[:10]}" if rank == 0 else None]
dist.broadcast_object_list(name, src=0)
ts = []
for k in range(5):
    dist.barrier()
    ts.append(eng.broadcast_model("actor", k % world, rank, world, f"{name[0]}_{k}"))
allt = [None] * world
dist.all_gather_object(allt, ts)
if rank == 0:
    t = min(max(r[k] for r in allt) for k in range(1, 5))
    print(f"{wl} actor {nb.value / 1e9:.3f} GB on {world} GPUs: {t * 1e3:.2f} ms "
          f"({nb.value / t / 1e9:.0f} GB/s of weights delivered per rank)", flush=True)
eng.close()
dist.destroy_process_group()
