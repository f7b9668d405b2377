"""Calibrate the decision clock's CostModel from measured B200 runs.

    python tools/calibrate.py [workload] [out.json]

The reference prices a decode step as decode_step_base * max(1, B / bs_max)
(genfuse.cpp:222-271) and a forward pass as per_layer_params * layers * tokens *
time_per_token_coeff (core.cpp:66-73). This tool measures both on one B200
through the engine's own execution (stage-barrier schedule, so decode and
scoring do not overlap), fits the constants, and reports how well the
calibrated decision clock predicts the measured stage times:

* decode: (rows, ms) of every decode step -> least-squares fit of
  base * max(1, B / bs_max) over a grid of bs_max;
* scoring: GPU busy time of the scoring batches / (sum over the three frozen
  models of per_layer_params * layers) / scored tokens -> time_per_token_coeff.

The JSON it writes is what configs.gen_config(..., calibrated=True) loads.
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402


PER_GPU = {"1.3b": 256, "8b": 64}  # bench.py --workload: prompts per GPU


def per_layer_params(d):  # core.cpp:56-60 (the reference's count; SwiGLU's third matrix is in the coefficient)
    return 4.0 * d.hidden * d.hidden + 2.0 * d.hidden * d.ffn


def fit_decode(rows, ms):
    rows = np.asarray(rows, np.float64)
    sec = np.asarray(ms, np.float64) * 1e-3
    best = None
    for bs_max in range(1, int(rows.max()) + 1):
        f = np.maximum(1.0, rows / bs_max)
        base = float(np.dot(f, sec) / np.dot(f, f))  # least squares for the scale
        err = float(np.sum((base * f - sec) ** 2))
        if best is None or err < best[0]:
            best = (err, base, bs_max)
    err, base, bs_max = best
    pred = base * np.maximum(1.0, rows / bs_max)
    return base, bs_max, float(np.sqrt(err / len(rows))), float(pred.sum()), float(sec.sum())


def main():
    wname = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
    out_path = Path(sys.argv[2]) if len(sys.argv) > 2 else None
    w = WORKLOADS[wname]
    if wname in PER_GPU:  # the bench's per-GPU batch (the full 1.3b batch needs a KV pool beyond one GPU)
        w = scaled(w, n_prompts=PER_GPU[wname])
    eng = Engine(w)
    batch = batch_for(w, eng.sched)
    cfg0 = gen_config(w, 1)
    runs = []
    for _ in range(3):
        runs.append(eng.execute(batch, cfg0, 0, token_mode="sample", schedule="stage_barrier", resident=True))
    out = runs[-1]
    base, bs_max, rmse, pred_dec, meas_dec = fit_decode(out.step_rows, out.step_ms)
    st = out.stats
    flops_params = sum(per_layer_params(d) * d.num_layers for d in (w.ref, w.critic, w.reward))
    coeff = st["infer_busy_seconds"] / (flops_params * st["infer_tokens"])
    cal = {"workload": wname, "decode_step_base": base, "bs_max": bs_max, "time_per_token_coeff": coeff,
           "decode_fit_rmse_s": rmse, "decode_steps": len(out.step_rows),
           "decode_measured_s": meas_dec, "decode_predicted_s": pred_dec,
           "infer_busy_s": st["infer_busy_seconds"], "infer_tokens": st["infer_tokens"]}
    # the calibrated decision clock vs the measured stage
    cfg = gen_config(w, 1, bs_max=bs_max, decode_step_base=base, time_per_token_coeff=coeff)
    serial = eng.sched.simulate_serial(batch, cfg)
    cal["clock_gen_end_s"] = serial.gen_end
    cal["clock_total_s"] = serial.total
    cal["measured_gen_s"] = st["gen_seconds"]
    cal["measured_wall_s"] = st["wall_seconds"]
    # R_t sweep with the calibrated model at G = 2, 4, 8 (the paper's workflow)
    sweeps = {}
    for G in (2, 4, 8):
        cg = gen_config(w, G, bs_max=bs_max, decode_step_base=base, time_per_token_coeff=coeff)
        bg = batch_for(w, eng.sched, n=w.n_prompts * G)
        sw = eng.sched.sweep_threshold(bg, cg)
        ratio, r_t, total = sw.curve[sw.best_index]
        sweeps[G] = {"best_ratio": ratio, "best_r_t": r_t, "best_fused_total_s": total,
                     "serial_total_s": sw.serial_total, "predicted_speedup": sw.serial_total / total}
    cal["sweep"] = sweeps
    eng.close()
    text = json.dumps(cal, indent=1)
    print(text)
    if out_path:
        out_path.write_text(text + "\n")


if __name__ == "__main__":
    main()
