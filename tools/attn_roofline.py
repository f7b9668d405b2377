"""Decode-attention roofline on a bench-shaped launch (gpt2s: H = KVH = 12, hd 64;
ATTN_SHAPE=8b: H 32, KVH 8, hd 128; 13b: H = KVH = 16, hd 128).

    python tools/attn_roofline.py [B] [mean_ctx]        # CUDA-event timing, L2 flushed per launch
    ncu --set full -k regex:attn_decode_mma -s 5 -c 1 python tools/attn_roofline.py ...

Algorithmic bytes per launch = K and V of every visible token of the layer
(2 x KVH x hd x 2 B per token) + q (B x H x hd x 2 B) — the same count bench.py's
probe uses. Prints one JSON line.
"""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
mean_ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 380
import os
# ATTN_SHAPE=8b: Llama-3-8B's GQA 32 / 8 heads of 128 (default: gpt2s MHA 12 x 64)
H, KVH, hd, PT = {"8b": (32, 8, 128, 64), "13b": (16, 16, 128, 64)}.get(os.environ.get("ATTN_SHAPE"), (12, 12, 64, 64))
L = int(os.environ.get("ATTN_L", "12"))  # layers per page (page bytes scale with L)
layer = min(5, L - 1)
lib = _lib.load()
if os.environ.get("ATTN_CUT") is not None:  # 0 whole splits (default), 1 128-token sub-chunks, -1 rule
    lib.fp_k_set_attn_cut(int(os.environ["ATTN_CUT"]))
g = torch.Generator().manual_seed(5)
ctx = (torch.rand(B, generator=g) * 2 * mean_ctx).clamp(min=1).to(torch.int32)  # uniform on [1, 2 mean)
maxp = (int(ctx.max()) + PT - 1) // PT
npages = B * maxp + 1
pool = torch.empty(npages, L, KVH, 2, PT, hd, device="cuda", dtype=torch.bfloat16).normal_()
bt = (torch.randperm(npages - 1)[: B * maxp] + 1).to(torch.int32).view(B, maxp).cuda()
slot = torch.arange(B, dtype=torch.int32, device="cuda")
ctx_d = ctx.cuda()
q = torch.randn(B, H, hd, device="cuda").to(torch.bfloat16)
out = torch.empty(B, H, hd, device="cuda", dtype=torch.bfloat16)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
clean = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB read after the flush: evicts its dirty lines


def flush_l2():
    # a 512 MB write leaves ~126 MB of dirty lines in L2, whose write-backs would be charged to the
    # timed launch; a 256 MB read afterwards evicts them, leaving L2 clean (and cold for the pool)
    flush.zero_()
    clean.sum()

p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
max_ctx = int(ctx.max())
ws = torch.zeros(int(lib.fp_k_attn_workspace_bytes(B, H, KVH, hd, max_ctx)), dtype=torch.uint8, device="cuda")
ns = (max_ctx + 63) // 64  # >= splits at any chunk >= 64
items_h = (C.c_int32 * (1 + B * ns))()
ctx_h = (C.c_int32 * B)(*[int(c) for c in ctx])
assert lib.fp_k_attn_items(ctx_h, B, H, KVH, hd, max_ctx, items_h) == 0
items = torch.tensor(list(items_h), dtype=torch.int32, device="cuda")


def run(st):
    r = lib.fp_k_attn_decode_ws(p(q), B, H, KVH, hd, p(pool), npages, L, layer, p(bt), maxp, p(slot), p(ctx_d),
                                p(items), max_ctx, p(ws), p(out), C.c_void_p(st))
    assert r == 0, r


s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        run(s.cuda_stream)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        run(s.cuda_stream)
torch.cuda.synchronize()
times = []
for _ in range(20):
    flush_l2()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1))
times.sort()
ms = times[len(times) // 2]
if "--trace" in sys.argv:
    import numpy as np
    tr = torch.zeros(4 * 148 * 12, dtype=torch.int64, device="cuda")
    lib.fp_k_attn_trace(p(tr))
    flush_l2()
    run(s.cuda_stream)
    torch.cuda.synchronize()
    lib.fp_k_attn_trace(None)
    t = tr.view(-1, 4).cpu().numpy()
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    pro = (t[:, 1] - t[:, 0]) / 1e3
    end = (t[:, 2] - t0) / 1e3
    print(f"trace: warps {len(t)}, entry spread {(t[:, 0].max() - t0) / 1e3:.2f} us, prologue med/max "
          f"{np.median(pro):.2f}/{pro.max():.2f} us, end min/med/max {end.min():.1f}/{np.median(end):.1f}/"
          f"{end.max():.1f} us (from first entry), units min/med/max {t[:, 3].min()}/{int(np.median(t[:, 3]))}/"
          f"{t[:, 3].max()}")
alg = float(ctx.sum()) * 2 * KVH * hd * 2 + B * H * hd * 2
print(json.dumps({"kernel": "attn_decode_mma_kernel<64,1>", "B": B, "ctx_sum": int(ctx.sum()),
                  "algorithmic_bytes": alg, "median_ms": ms, "achieved_GBps": alg / (ms / 1e3) / 1e9,
                  "note": "one graph-replayed launch (fp_k_attn_decode_ws), CUDA events, L2 flushed "
                          "(512 MiB write, then a 256 MiB read so no dirty line is written back during the launch) "
                          "before each of 20 timed launches; median"}))
