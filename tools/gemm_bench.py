"""Microbenchmark of the tcgen05 GEMM launchers (CUDA events, warm, L2 flushed between reps).

    python tools/gemm_bench.py                 # the decode / prefill shape table
    python tools/gemm_bench.py KIND M N K      # one shape (for an ncu capture)
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib  # noqa: E402

lib = _lib.load()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, reps=20):
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2] * 1000  # us


def run(kind, M, N, K):
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    if kind == "bf16":
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        f = lambda: lib.fp_k_gemm_bf16(p(W), N, K, p(X), M, p(out), N, None)  # noqa: E731
    elif kind == "f32":
        s = lib.fp_k_gemm_splits(N, K)
        out = torch.empty(s, M, N, device="cuda")
        f = lambda: lib.fp_k_gemm_f32(p(W), N, K, p(X), M, p(out), s, None)  # noqa: E731
    elif kind == "swiglu":
        out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        f = lambda: lib.fp_k_gemm_swiglu(p(W), N // 2, K, p(X), M, p(out), None)  # noqa: E731
    us = timeit(f)
    wbytes = N * K * 2
    flops = 2 * M * N * K
    print(f"{kind:7s} M={M:5d} N={N:6d} K={K:5d}: {us:8.2f} us  W {wbytes/us/1e3:7.1f} GB/s  {flops/us/1e6:7.1f} TF/s",
          flush=True)


if len(sys.argv) == 5:
    run(sys.argv[1], *map(int, sys.argv[2:]))
    sys.exit(0)
for kind, N, K in (("bf16", 2304, 768), ("swiglu", 6144, 768), ("f32", 768, 3072), ("f32", 768, 768),
                   ("bf16", 6144, 768), ("bf16", 12288, 4096)):
    for M in (16, 64, 128, 256, 512):
        run(kind, M, N, K)
for M in (2048, 8192, 16384):
    run("bf16", M, 6144, 768)
    run("bf16", M, 2304, 768)
