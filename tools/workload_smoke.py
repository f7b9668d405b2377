"""Run the larger SURVEY workloads' model shapes end to end on one GPU (few prompts):
1.3B (d 2048, hd 128) and Llama-3-8B shape (GQA 32/8, hd 128, V 128256).

    python tools/workload_smoke.py [names...]
"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

for name in sys.argv[1:] or ["1.3b", "8b"]:
    w = scaled(WORKLOADS[name], n_prompts=64, max_new=512 if name == "8b" else 256)
    t0 = time.perf_counter()
    eng = Engine(w, max_samples=64, max_live=64)
    batch = batch_for(w, eng.sched)
    for mode in ("forced", "sample"):
        out = eng.execute(batch, gen_config(w, 1, calibrated=False), 0, token_mode=mode, schedule="fused",
                          claim_tokens=16384)
        x = out.experience
        finite = all(np.isfinite(getattr(x, k)).all() for k in ("logp_actor", "logp_ref", "values", "adv", "ret"))
        st = out.stats
        print(f"{name} {mode}: {len(batch)} samples, {st['decode_steps']} steps, gen {st['gen_seconds']:.3f} s, "
              f"wall {st['wall_seconds']:.3f} s, finite {finite}, mean logp {float(x.logp_actor.mean()):.3f}, "
              f"mean kl {float(x.kl.mean()):.4f}", flush=True)
    eng.close()
    print(f"{name}: total {time.perf_counter() - t0:.1f} s", flush=True)
