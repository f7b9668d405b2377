"""Fused-schedule wall time vs claim_max_live (scoring on a generating GPU only
once its live decode batch is at most this many rows; 0 = always), 1 GPU.

    python tools/claim_live_sweep.py [gpt2s|1.3b|8b] [values ...]
"""
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
    vals = [int(v) for v in sys.argv[2:]] or [0, 16, 32, 64, 128]
    w = WORKLOADS[name]
    if name == "1.3b":
        w = scaled(w, n_prompts=256)
    eng = Engine(w)
    batch = batch_for(w, eng.sched)
    cfg = gen_config(w, 1)
    eng.execute(batch, cfg, 0, token_mode="sample", schedule="fused", resident=True)  # warm-up / graphs

    def wall(**kw):
        ts = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.execute(batch, cfg, 0, token_mode="sample", resident=True, **kw)
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts)

    base = wall(schedule="stage_barrier")
    print(f"{name}: stage barrier {base:.3f} s")
    for v in vals:
        t = wall(schedule="fused", claim_max_live=v)
        print(f"  fused, claim_max_live {v:4d}: {t:.3f} s ({base / t:.3f}x)")


if __name__ == "__main__":
    main()
