"""Scoring-shape kernels timed alone (CUPTI device time, mean of 20, inputs
L2-resident as in the packed forward): the per-layer GEMMs of the scoring
models at M = 8192 packed tokens, the RMSNorm and the attention.

    python tools/scoring_gemm_probe.py [gpt2s|1.3b|8b]
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib, configs  # noqa: E402

lib = _lib.load()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def timeit(fn, reps=20):
    """Mean device duration of the kernels fn launches (CUPTI via torch.profiler; each call synchronised, so
    no PDL overlap with a neighbour is counted, and the host launch latency is not)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
            torch.cuda.synchronize()
    ts = [e.device_time for e in prof.events() if e.device_time > 0 and "Memcpy" not in e.name]
    return sum(ts) / reps  # us


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
    D = configs.WORKLOADS[name].ref
    M, d, F = 8192, D.hidden, D.ffn
    qkv = (D.num_heads + 2 * D.num_kv_heads) * D.head_dim
    ao = D.num_heads * D.head_dim
    s = None
    X = torch.randn(M, max(d, F, ao), device="cuda").to(torch.bfloat16)
    rows = []
    for kind, N, K in (("qkv bf16", qkv, d), ("o resid", d, ao), ("gate/up swiglu", 2 * F, d), ("down resid", d, F)):
        W = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
        Xk = X[:, :K].contiguous()
        if "resid" in kind:
            out = torch.zeros(M, N, device="cuda")
            f = lambda: lib.fp_k_gemm_f32_residual(p(W), N, K, p(Xk), M, p(out), s)  # noqa: E731
        elif "swiglu" in kind:
            out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
            f = lambda: lib.fp_k_gemm_swiglu(p(W), N // 2, K, p(Xk), M, p(out), s)  # noqa: E731
        else:
            out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            f = lambda: lib.fp_k_gemm_bf16(p(W), N, K, p(Xk), M, p(out), N, s)  # noqa: E731
        us = timeit(f)
        rows.append((kind, us, 2 * M * N * K / us / 1e6))
    x = torch.randn(M, d, device="cuda")
    g = torch.ones(d, device="cuda")
    y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    us = timeit(lambda: lib.fp_k_rms_norm_rows(p(x), p(g), p(y), M, d, s))
    # the layer as the packed forward enqueues it (back to back, PDL between the
    # GEMMs and norms), 12 layers, timed with events around the whole chain
    lens = [300] * (M // 300)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    Mq = int(cu[-1])
    H, KVH, hd = D.num_heads, D.num_kv_heads, D.head_dim
    q = torch.randn(Mq, H, hd, device="cuda").bfloat16()
    kk = torch.randn(Mq, KVH, hd, device="cuda").bfloat16()
    vv = torch.randn(Mq, KVH, hd, device="cuda").bfloat16()
    att = torch.empty(M, ao, device="cuda", dtype=torch.bfloat16)
    cud = torch.from_numpy(cu).cuda()
    cuh = cu.ctypes.data_as(C.POINTER(C.c_int32))
    Wq = (torch.randn(qkv, d, device="cuda") * d ** -0.5).bfloat16()
    Wo = (torch.randn(d, ao, device="cuda") * ao ** -0.5).bfloat16()
    Wgu = (torch.randn(2 * F, d, device="cuda") * d ** -0.5).bfloat16()
    Wd = (torch.randn(d, F, device="cuda") * F ** -0.5).bfloat16()
    h = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    qkvo = torch.empty(M, qkv, device="cuda", dtype=torch.bfloat16)
    act = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
    ta = timeit(lambda: lib.fp_k_attn_varlen(p(q), p(kk), p(vv), H, KVH, hd, cuh, p(cud), len(lens), p(att), s))

    def layer():
        lib.fp_k_rms_norm_rows(p(x), p(g), p(h), M, d, s)
        lib.fp_k_gemm_bf16(p(Wq), qkv, d, p(h), M, p(qkvo), qkv, s)
        lib.fp_k_gemm_f32_residual(p(Wo), d, ao, p(att), M, p(x), s)
        lib.fp_k_rms_norm_rows(p(x), p(g), p(h), M, d, s)
        lib.fp_k_gemm_swiglu(p(Wgu), F, d, p(h), M, p(act), s)
        lib.fp_k_gemm_f32_residual(p(Wd), d, F, p(act), M, p(x), s)

    for _ in range(2):
        layer()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(12):
        layer()
    e1.record()
    torch.cuda.synchronize()
    chain = e0.elapsed_time(e1) * 1000 / 12
    alone = sum(r[1] for r in rows) + 2 * us
    print(f"{name} M={M}:")
    for kind, us_, tf in rows:
        print(f"  {kind:16s} {us_:8.1f} us {tf:7.0f} TF/s")
    print(f"  rms_norm_rows    {us:8.1f} us {M * d * 6 / us / 1e3:7.0f} GB/s")
    print(f"  attention        {ta:8.1f} us (L = 300 x {len(lens)})")
    print(f"  layer without attention: chained (events, PDL) {chain:.1f} us vs sum of kernels alone {alone:.1f} us")


if __name__ == "__main__":
    main()
