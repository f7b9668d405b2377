"""SM-pair (cta_group::2) packed GEMM vs the one-SM persistent kernel vs the automatic
choice (fp_k_set_pair_gemm 0 / 1 / -1): bits and time.

    python tools/pair_gemm_check.py [gpt2s|1.3b|8b]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib, configs  # noqa: E402

lib = _lib.load()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def kernel_us(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            fn()
            torch.cuda.synchronize()
    ts = [e.device_time for e in prof.events() if e.device_time > 0 and "Memcpy" not in e.name]
    return sum(ts) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
    D = configs.WORKLOADS[name].ref
    M, d, F = 8192, D.hidden, D.ffn
    ao = D.num_heads * D.head_dim
    X = (torch.rand(M, max(d, F, ao), device="cuda") * 2 - 1).to(torch.bfloat16)
    for kind, N, K in (("o resid", d, ao), ("gate/up swiglu", 2 * F, d), ("down resid", d, F)):
        W = ((torch.rand(N, K, device="cuda") * 2 - 1) * K ** -0.5).to(torch.bfloat16)
        Xk = X[:, :K].contiguous()
        r0 = torch.randn(M, N, device="cuda")
        outs, ts = [], []
        for pair in (0, 1, -1):
            lib.fp_k_set_pair_gemm(pair)
            if "resid" in kind:
                o = r0.clone()
                f = lambda: lib.fp_k_gemm_f32_residual(p(W), N, K, p(Xk), M, p(o), None)  # noqa: E731
                f()
                torch.cuda.synchronize()
                outs.append(o.clone())
            else:
                o = torch.full((M, N // 2), float("nan"), device="cuda", dtype=torch.bfloat16)
                f = lambda: lib.fp_k_gemm_swiglu(p(W), N // 2, K, p(Xk), M, p(o), None)  # noqa: E731
                f()
                torch.cuda.synchronize()
                outs.append(o.clone())
            ts.append(kernel_us(f))
        lib.fp_k_set_pair_gemm(-1)
        same = torch.equal(outs[0], outs[1])
        diff = (outs[0].float() - outs[1].float()).abs().max().item()
        fl = 2 * M * N * K
        extra = ""
        if len(ts) > 2:
            extra = f", auto {ts[2]:.1f} us (same bits {torch.equal(outs[0], outs[2])})"
        print(f"{name} {kind} M={M} N={N} K={K}: one-SM {ts[0]:.1f} us ({fl / ts[0] / 1e6:.0f} TF/s), "
              f"pair {ts[1]:.1f} us ({fl / ts[1] / 1e6:.0f} TF/s){extra}; bit-identical {same} (max |diff| {diff:.3g})")


if __name__ == "__main__":
    main()
