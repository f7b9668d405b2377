"""Per-kernel device time of one stage-barrier bench step on 1 B200, split by
stream (decode vs scoring), from CUPTI (torch.profiler) — where the scoring
stage's time goes (inference_roofline's denominator).

    python tools/infer_breakdown.py [gpt2s|1.3b] [out.json]
"""
import json
import sys
from collections import defaultdict
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2409_13221_b200.configs import WORKLOADS, batch_for, gen_config, scaled  # noqa: E402
from paper_2409_13221_b200.engine import Engine  # noqa: E402


def short(name: str) -> str:
    for k in ("attn_prefill_kernel", "attn_varlen_kernel", "attn_decode", "tc_gemm_kernel", "vocab", "add_norm",
              "embed", "assemble", "postprocess", "rope", "topk", "chain"):
        if k in name:
            if k == "tc_gemm_kernel":
                epi = name.split("fpk::", 2)[-1].split("<")[0] if "fpk::" in name else "?"
                return f"gemm[{epi}]"
            return k
    return name[:60]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
    w = WORKLOADS[name]
    if name == "1.3b":
        w = scaled(w, n_prompts=256)
    eng = Engine(w)
    batch = batch_for(w, eng.sched)
    cfg = gen_config(w, 1)
    eng.execute(batch, cfg, 0, token_mode="sample", schedule="stage_barrier", resident=True)  # warm-up
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        out = eng.execute(batch, cfg, 0, token_mode="sample", schedule="stage_barrier", resident=True)
        torch.cuda.synchronize()
    by_stream = defaultdict(lambda: defaultdict(lambda: [0, 0.0]))
    spans = defaultdict(list)
    for e in prof.events():
        if e.device_type != torch.autograd.DeviceType.CUDA or e.device_time <= 0:
            continue
        spans[getattr(e, "device_resource_id", 0)].append((e.time_range.start, e.time_range.end))
        s = by_stream[getattr(e, "device_resource_id", 0)][short(e.name)]
        s[0] += 1
        s[1] += e.device_time / 1e3  # ms
    res = {"workload": name, "stats": out.stats,
           "streams": {}}
    for sid, ks in by_stream.items():
        tot = sum(v[1] for v in ks.values())
        res["streams"][str(sid)] = {"total_ms": tot, "kernels": {k: {"launches": v[0], "ms": v[1]}
                                                               for k, v in sorted(ks.items(), key=lambda x: -x[1][1])}}
        iv = sorted(spans[sid])
        busy, cur_s, cur_e = 0.0, iv[0][0], iv[0][1]
        for a, b in iv[1:]:
            if a > cur_e:
                busy += cur_e - cur_s
                cur_s, cur_e = a, b
            else:
                cur_e = max(cur_e, b)
        busy += cur_e - cur_s
        span = iv[-1][1] - iv[0][0]
        res["streams"][str(sid)].update(span_ms=span / 1e3, busy_union_ms=busy / 1e3)
        print(f"stream {sid}: kernel-time sum {tot:.1f} ms, first-to-last span {span / 1e3:.1f} ms, "
              f"union of kernel intervals {busy / 1e3:.1f} ms")
        for k, v in sorted(ks.items(), key=lambda x: -x[1][1])[:14]:
            print(f"   {k:40s} {v[0]:7d} launches {v[1]:9.2f} ms ({v[1] / tot:.1%})")
    # all streams but the busiest-by-launch-count decode stream: the scoring streams together
    dec = max(by_stream, key=lambda k: sum(v[0] for v in by_stream[k].values()))
    iv = sorted(x for sid, xs in spans.items() if sid != dec for x in xs)
    if iv:
        busy, cs, ce = 0.0, iv[0][0], iv[0][1]
        for a, b in iv[1:]:
            if a > ce:
                busy += ce - cs
                cs, ce = a, b
            else:
                ce = max(ce, b)
        busy += ce - cs
        res["scoring_union_ms"] = busy / 1e3
        res["scoring_span_ms"] = (iv[-1][1] - iv[0][0]) / 1e3
        print(f"scoring streams together: union {busy / 1e3:.1f} ms, span {(iv[-1][1] - iv[0][0]) / 1e3:.1f} ms")
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_text(json.dumps(res, indent=1, default=str))


if __name__ == "__main__":
    main()
