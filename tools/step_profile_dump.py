"""Per-decode-step (rows, GPU ms) of one gpt2s bench step (stage barrier and
fused), for the time-vs-batch-size breakdown in DESIGN.md.

    python tools/step_profile_dump.py out.json
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

w = WORKLOADS["gpt2s"]
eng = Engine(w)
batch = batch_for(w, eng.sched)
res = {}
for sched in ("stage_barrier", "fused", "stage_barrier", "fused"):
    out = eng.execute(batch, gen_config(w, 1), 0, token_mode="sample", schedule=sched, resident=True)
    res[sched] = {"rows": out.step_rows.tolist(), "ms": out.step_ms.tolist(),
                  "gen_seconds": out.stats["gen_seconds"], "infer_busy": out.stats["infer_busy_seconds"],
                  "wall": out.stats["wall_seconds"]}
Path(sys.argv[1]).write_text(json.dumps(res))
