"""In-step timeline of one decode step (globaltimer stamps from every GEMM CTA and
decode-attention warp / team CTA; the other kernels show up as gaps).

    python tools/step_trace.py run STEP [out.json]    # gpt2s bench batch, stage barrier, traces decode step STEP
    python tools/step_trace.py show out.json
"""
import json
import os
import subprocess
import sys

import numpy as np

DETAIL = '--detail' in sys.argv

KIND = {0: "gemm", 1: "attn", 2: "attn-team", 3: "chain"}
# decode_chain stamps (16 per CTA): see csrc/kernels/chain.cu
CHAIN = [(1, "P0 acc"), (2, "P0 arrive"), (3, "P1 wait"), (4, "P1 arrive"), (14, "P2 act-in"), (5, "P2 acc"),
         (6, "P2 arrive"), (7, "P3 wait"), (8, "P3 acc"), (9, "P3 arrive"), (10, "P4 wait"), (11, "P4 arrive"),
         (15, "P5 act-in"), (12, "P5 acc"), (13, "P5 end")]


def run(step, out):
    env = dict(os.environ, FUSEPLAN_TRACE_STEP=str(step), FUSEPLAN_TRACE_OUT=out)
    code = ("import sys; sys.path.insert(0, '.');"
            "from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config;"
            "from paper_2409_13221_b200.engine import Engine;"
            "w = WORKLOADS['gpt2s']; e = Engine(w); b = batch_for(w, e.sched);"
            "e.execute(b, gen_config(w, 1), 0, token_mode='sample', schedule='stage_barrier', resident=True)")
    subprocess.run([sys.executable, "-c", code], env=env, check=True)
    show(out)


def show(path):
    d = json.load(open(path))
    rows = []
    for i, L in enumerate(d["launches"]):
        x = L["data"]
        if L["kind"] == 0:  # 8 words per CTA: entry, setup, first_full, last_full, acc, epi_done
            cta = [x[k:k + 8] for k in range(0, len(x), 8)]
            cta = [c for c in cta if c[0] > 0]
            beg, end = min(c[0] for c in cta), max(max(c[5], c[4], c[0]) for c in cta)
            first = sorted(c[2] - c[0] for c in cta if c[2])
            extra = f"ctas {len(cta):4d}, first-data median {first[len(first) // 2] / 1e3:5.2f} us" if first else ""
        elif L["kind"] == 3:  # decode_chain: 16 stamps per CTA
            cta = [x[k:k + 16] for k in range(0, len(x), 16)]
            beg = min(c[0] for c in cta if c[0])
            end = max(max(c) for c in cta)
            extra = f"ctas {len(cta):4d}"
            if DETAIL:
                for col, nm in CHAIN:
                    v = np.array([c[col] for c in cta if c[col] > 0], dtype=np.float64)
                    if len(v):
                        extra += f"\n      {nm:10s} " + " ".join(f"{(q - beg) / 1e3:6.2f}" for q in np.percentile(v, [0, 50, 100]))
        else:  # 4 words per warp / CTA: entry, loop-begin, end, units
            w = [x[k:k + 4] for k in range(0, len(x), 4)]
            w = [v for v in w if v[0] > 0]
            beg, end = min(v[0] for v in w), max(v[2] for v in w)
            extra = f"units {len(w):5d} (warps/CTAs)"
        if L["kind"] == 2 and DETAIL:  # team CTAs: entry, wait return, end, first item done
            for nm, col in (("entry", 0), ("wait", 1), ("first", 3), ("end", 2)):
                v = np.array([c[col] for c in w if c[col] > 0], dtype=np.float64)
                extra += f"\n      {nm:5s} " + " ".join(f"{(q - beg) / 1e3:6.2f}" for q in np.percentile(v, [0, 10, 50, 90, 100]))
        rows.append((beg, end, KIND[L["kind"]], extra))
    t0 = rows[0][0]
    print(f"decode step: B={d['B']} max_ctx={d['max_ctx']} ctx_sum={d['ctx_sum']:.0f}")
    prev = None
    eff = {}
    for beg, end, kind, extra in rows:
        # launches overlap under PDL (CTAs start early and wait): the effective
        # time of a launch is from the previous traced launch's end to its own end
        e = (end - max(beg, prev if prev is not None else beg)) / 1e3
        print(f"  {kind:9s} start {(beg - t0) / 1e3:8.2f} us  end {(end - t0) / 1e3:8.2f} us  "
              f"effective {e:6.2f} us  {extra}")
        eff[kind] = eff.get(kind, 0.0) + e
        prev = end
    total = (rows[-1][1] - t0) / 1e3
    print(f"  span {total:.1f} us; effective " + ", ".join(f"{k} {v:.1f} us" for k, v in eff.items()) +
          " (gemm includes the untraced add_norm / embed / finalize kernels between launches)")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/step_trace.json")
    else:
        show(sys.argv[2])
