"""Decode-step GPU time vs live batch size for the bench workload (1 GPU)."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402

w = WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "gpt2s"]
sched = sys.argv[2] if len(sys.argv) > 2 else "stage_barrier"
eng = Engine(w)
batch = batch_for(w, eng.sched)
cfg = gen_config(w, 1)
for _ in range(2):
    out = eng.execute(batch, cfg, 0, token_mode="sample", schedule=sched, resident=True)
rows, ms = out.step_rows, out.step_ms
print(f"{w.name} {sched}: steps {len(rows)} total decode {ms.sum():.1f} ms, gen {out.stats['gen_seconds']*1e3:.1f} ms")
for lo, hi in ((1, 8), (9, 32), (33, 64), (65, 128), (129, 256), (257, 512)):
    sel = (rows >= lo) & (rows <= hi)
    if sel.any():
        print(f"  B in [{lo:3d},{hi:3d}]: {sel.sum():4d} steps, mean {ms[sel].mean():.3f} ms, total {ms[sel].sum():7.1f} ms")
# linear fit ms = a + b * B (the decision clock's decode_step_base / bs_max plateau)
A = np.vstack([np.ones_like(rows, dtype=np.float64), rows.astype(np.float64)]).T
coef, *_ = np.linalg.lstsq(A, ms.astype(np.float64), rcond=None)
print(f"  fit: step_ms = {coef[0]:.4f} + {coef[1]*1e3:.4f}e-3 * B")
