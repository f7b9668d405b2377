"""One small experience-collection pass for compute-sanitizer (racecheck /
synccheck / memcheck): toy workload, 8 prompts, every token mode, both
schedules, and the decode-chain kernel (FUSEPLAN_DECODE_CHAIN=512).

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

w = scaled(WORKLOADS["toy"], n_prompts=8, max_new=40, prompt_len=16)
eng = Engine(w, device=0)
batch = batch_for(w, eng.sched)
for mode, sched in (("forced", "fused"), ("greedy", "stage_barrier"), ("sample", "fused")):
    out = eng.execute(batch, gen_config(w, 1), 0, token_mode=mode, schedule=sched, claim_tokens=128)
    print(mode, sched, out.stats["decode_steps"], "steps", flush=True)
out = eng.execute(batch, gen_config(w, 1), 0, token_mode="sample", top_k=8, top_p=0.9)
print("filtered", out.stats["decode_steps"], flush=True)
eng.close()
os.environ["FUSEPLAN_DECODE_CHAIN"] = "512"
eng = Engine(w, device=0)
out = eng.execute(batch, gen_config(w, 1), 0, token_mode="sample", schedule="fused")
print("chain", out.stats["decode_steps"], flush=True)
eng.close()
