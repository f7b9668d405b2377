"""Per-decode-step (rows, visible context, GPU ms) and scoring totals of one
bench step on 1 B200, stage barrier and fused — the measurements the R_t
chooser (tools/rt_chooser.py) fits its step and sharing model to, and the
time-vs-batch-size breakdown in DESIGN.md §8.

    python tools/step_profile_dump.py gpt2s|1.3b|8b out.json
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

name = sys.argv[1]
w = WORKLOADS[name]
pool = 0
if name == "1.3b":
    w = scaled(w, n_prompts=256)  # the bench's per-GPU batch
if name == "8b":
    w = scaled(w, n_prompts=512)  # configs[3]'s per-GPU batch, KV-gated as bench.py --kv-pool-gb 96
    pool = int(96e9)
eng = Engine(w, kv_pool_bytes=pool)
batch = batch_for(w, eng.sched)
cfg = gen_config(w, 1)
if pool:
    page = 64 * eng.kv_bytes_per_token()
    cfg.cluster.kv_capacity_per_instance = (pool - w.n_prompts * page) * 4.0 * w.actor.num_layers * \
        w.actor.hidden / eng.kv_bytes_per_token()
res = {"workload": name, "n": len(batch), "prompt_len": w.prompt_len,
       "lengths": [b.target_output_len for b in batch], "kv_capacity": cfg.cluster.kv_capacity_per_instance,
       "kv_bytes": [b.kv_bytes for b in batch]}
for rep in range(1 if name == "8b" else 2):
    for sched in ("stage_barrier", "fused"):
        out = eng.execute(batch, cfg, 0, token_mode="sample", schedule=sched, resident=True)
        if rep == 0 and name != "8b":
            continue  # warm-up (graphs captured; 8b: one pass, its steps dominate the capture cost)
        res[sched] = {"rows": out.step_rows.tolist(), "ms": out.step_ms.tolist(), "ctx": out.step_ctx.tolist(),
                      "gen_seconds": out.stats["gen_seconds"], "infer_busy": out.stats["infer_busy_seconds"],
                      "infer_tokens": out.stats["infer_tokens"], "wall": out.stats["wall_seconds"],
                      "finish": out.finish_seconds.tolist()}
Path(sys.argv[2]).write_text(json.dumps(res))
