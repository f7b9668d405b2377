"""Scoring-attention probe: time fp_k_attn_varlen (tcgen05) and fp_k_attn_varlen_mma
(mma.sync) on one packed scoring batch of each workload's real length mix
(prompt + Zipf response lengths, packed to ~8192 tokens like Engine::infer),
beside the SwiGLU GEMM of the same M for scale.

    python tools/varlen_probe.py [gpt2s|1.3b|8b ...] [L=<uniform length>]   # on a B200 (gpurun)

Kernel times are CUPTI device durations. Reports causal FLOPs (4 * sum(L^2 / 2) * H * hd) per second.
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib, configs  # noqa: E402

lib = _lib.load()


def p(t):
    return C.c_void_p(t.data_ptr())


def timeit(fn, n=30, reps=3):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / n)
    return best  # ms, best of `reps` means


def kernel_us(fn, name_part, n=20):
    """Average device duration (us) of the kernels whose name contains name_part (CUPTI via torch.profiler):
    the C-ABI call synchronises on the host, so event timing would include that round trip."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
    ts = [e.device_time for e in prof.events() if name_part in e.name and e.device_time > 0]
    return sum(ts) / max(len(ts), 1) / 1e3 if ts else float("nan")  # ms


def packed_lengths(w, cap=8192):
    out = configs.zipf_lengths(w.n_prompts, w.max_new, w.zipf_s, w.zipf_lo, w.length_seed)
    lens, tot = [], 0
    for r in out:
        L = w.prompt_len + r
        if tot + L > cap and lens:
            break
        lens.append(L)
        tot += L
    return lens


def main():
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    args = [a for a in sys.argv[1:] if not a.startswith("L=")]
    uni = [int(a[2:]) for a in sys.argv[1:] if a.startswith("L=")]
    names = args or ["gpt2s", "1.3b", "8b"]
    for name in names:
        w = configs.WORKLOADS[name]
        D = w.ref
        H, KVH, hd, d, F = D.num_heads, D.num_kv_heads, D.head_dim, D.hidden, D.ffn
        lens = [uni[0]] * (8192 // uni[0]) if uni else packed_lengths(w)
        cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        M = int(cu[-1])
        q = torch.randn(M, H, hd, device="cuda").bfloat16()
        k = torch.randn(M, KVH, hd, device="cuda").bfloat16()
        v = torch.randn(M, KVH, hd, device="cuda").bfloat16()
        out = torch.empty(M, H, hd, device="cuda", dtype=torch.bfloat16)
        cud = torch.from_numpy(cu).cuda()
        cuh = cu.ctypes.data_as(C.POINTER(C.c_int32))
        fl = sum(4 * L * L / 2 * H * hd for L in lens)
        ta = kernel_us(lambda: lib.fp_k_attn_varlen(p(q), p(k), p(v), H, KVH, hd, cuh, p(cud), len(lens), p(out), s),
                       "attn_prefill_kernel")
        tm = kernel_us(lambda: lib.fp_k_attn_varlen_mma(p(q), p(k), p(v), H, KVH, hd, cuh, p(cud), len(lens), p(out),
                                                        s), "attn_varlen_kernel")
        W = torch.randn(2 * F, d, device="cuda").bfloat16()
        X = torch.randn(M, d, device="cuda").bfloat16()
        o = torch.empty(M, F, device="cuda", dtype=torch.bfloat16)
        tg = timeit(lambda: lib.fp_k_gemm_swiglu(p(W), F, d, p(X), M, p(o), s))
        print(f"{name}: H{H}/{KVH} hd{hd} {len(lens)} seqs M={M} (L mean {np.mean(lens):.0f} max {max(lens)}): "
              f"tcgen05 {ta * 1e3:.1f} us = {fl / ta / 1e9:.0f} TF/s | mma.sync {tm * 1e3:.1f} us = "
              f"{fl / tm / 1e9:.0f} TF/s | swiglu GEMM {tg * 1e3:.1f} us = {2 * M * 2 * F * d / tg / 1e9:.0f} TF/s")




def trace(name="gpt2s", L="128"):
    L = int(L)
    """CTA 0's per-block event times (us from its first stamp) of one launch."""
    w = configs.WORKLOADS[name]
    D = w.ref
    H, KVH, hd = D.num_heads, D.num_kv_heads, D.head_dim
    lens = [L] * (8192 // L)
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    M = int(cu[-1])
    q = torch.randn(M, H, hd, device="cuda").bfloat16()
    k = torch.randn(M, KVH, hd, device="cuda").bfloat16()
    v = torch.randn(M, KVH, hd, device="cuda").bfloat16()
    out = torch.empty(M, H, hd, device="cuda", dtype=torch.bfloat16)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    cud = torch.from_numpy(cu).cuda()
    buf = torch.zeros(8 * 64, dtype=torch.int64, device="cuda")
    lib.fp_k_attn_varlen(p(q), p(k), p(v), H, KVH, hd, cu.ctypes.data_as(C.POINTER(C.c_int32)), p(cud), len(lens),
                         p(out), s)
    lib.fp_k_attn_prefill_trace(p(buf))
    lib.fp_k_attn_varlen(p(q), p(k), p(v), H, KVH, hd, cu.ctypes.data_as(C.POINTER(C.c_int32)), p(cud), len(lens),
                         p(out), s)
    lib.fp_k_attn_prefill_trace(None)
    torch.cuda.synchronize()
    t = buf.view(8, 64).cpu().numpy()
    t0 = t[t > 0].min()
    names = ["K load", "S issued", "PV issued", "sm: S ready", "sm: max done / P buffer free", "sm: P written",
             "sm: item done", "sm: S in registers"]
    print(f"{name} L={L}: CTA 0 timeline (us)")
    for g in range(24):
        row = " ".join(f"{(t[kk, g] - t0) / 1e3:7.2f}" if t[kk, g] else "      -" for kk in range(8))
        print(f"  g={g:2d} {row}")
    print("  cols:", " | ".join(names))


if __name__ == "__main__":
    if "trace" in sys.argv:
        trace(*(a for a in sys.argv[1:] if a != "trace"))
    else:
        main()
