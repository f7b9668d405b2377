"""Per-kernel time of one decode step at a fixed live batch size (gpt2s dims).

    python tools/decode_breakdown.py run B [steps]          # executes B prompts x `steps` tokens
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file X.csv \
        python tools/decode_breakdown.py run B [steps]
    python tools/decode_breakdown.py report X.csv B [steps]  # aggregate the decode kernels per step
"""
import csv
import re
import sys
from collections import defaultdict

sys.path.insert(0, ".")


def run(B, steps):
    from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled
    from paper_2409_13221_b200.engine import Engine
    w = scaled(WORKLOADS["gpt2s"], n_prompts=B)
    eng = Engine(w, max_samples=B, max_live=B)
    batch = batch_for(w, eng.sched, lengths=[steps] * B)
    out = eng.execute(batch, gen_config(w, 1), 0, token_mode="sample", schedule="stage_barrier", resident=True)
    print(f"B={B} steps={len(out.step_rows)} decode {out.step_ms.sum():.2f} ms "
          f"({out.step_ms.mean():.3f} ms/step, last {out.step_ms[-4:].mean():.3f})")


def short(name):
    name = re.sub(r"\(anonymous namespace\)::|<?unnamed>::", "", name)
    name = re.sub(r"\(.*", "", name)
    name = re.sub(r"^void ", "", name)
    m = re.match(r"(?:fpk::)?(?:\(anonymous namespace\)::)?([\w:]+)(<.*>)?", name)
    base = m.group(1) if m else name
    if m and m.group(2):
        args = m.group(2)
        epi = re.search(r"Epi\w+(<[^>]*>)?", args)
        bn = re.match(r"<(\d+)", args)
        base += f"<{bn.group(1) if bn else ''}{',' + epi.group(0) if epi else ''}>"
    return base


def report(path, B, steps):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        v = v / 1000.0 if r[ui] in ("nsecond", "ns") else v if r[ui] in ("usecond", "us") else v * 1000.0
        per[short(r[ki])].append(v)
    tot = 0.0
    print(f"{'kernel':60s} {'launches':>8s} {'us/launch':>10s} {'us/step':>9s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        s = sum(v) / max(steps, 1)
        tot += s
        print(f"{k:60s} {len(v):8d} {sum(v) / len(v):10.2f} {s:9.2f}")
    print(f"{'total (all kernels, per decode step)':60s} {'':8s} {'':10s} {tot:9.2f}")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 32)
    else:
        report(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]) if len(sys.argv) > 4 else 32)
