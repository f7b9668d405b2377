"""Fused schedule on one B200: step time vs claim_max_live (when scoring may overlap decode).

    python tools/claim_sweep.py [values...]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

vals = [int(v) for v in sys.argv[1:]] or [0, 384, 256, 192, 128, 96, 64]
w = WORKLOADS["gpt2s"]
eng = Engine(w)
batch = batch_for(w, eng.sched)
cfg = gen_config(w, 1)
prompts = eng.synthetic_prompts(len(batch), 7)
for v in vals:
    ts = []
    for k in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = eng.execute(batch, cfg, 0, token_mode="sample", schedule="fused", prompts=prompts, resident=True,
                          claim_max_live=v)
        torch.cuda.synchronize()
        if k:
            ts.append(time.perf_counter() - t0)
    st = out.stats
    print(f"claim_max_live={v:4d}: step {1e3 * min(ts):7.1f} ms ({len(batch) / min(ts):6.1f} samples/s), "
          f"gen {1e3 * st['gen_seconds']:6.1f} ms, decode {1e3 * st['decode_gpu_seconds']:6.1f} ms, "
          f"infer busy {1e3 * st['infer_busy_seconds']:6.1f} ms", flush=True)
eng.close()
