"""Per-CTA tile timeline of the persistent packed-forward GEMM
(gemm_persist.cuh; globaltimer stamps through fp_k_gemm_trace): for each
CTA's tiles, when its MMAs started / were all issued, when the epilogue saw the
accumulator and when it finished.

    python tools/gemm_persist_trace.py [gpt2s|1.3b|8b]
"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib, configs  # noqa: E402

lib = _lib.load()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731


def run(kind, N, K, M, fn):
    buf = torch.zeros(148 * 8 * 4, dtype=torch.int64, device="cuda")
    fn()
    torch.cuda.synchronize()
    lib.fp_k_gemm_trace(p(buf))
    fn()
    lib.fp_k_gemm_trace(None)
    torch.cuda.synchronize()
    t = buf.view(148, 8, 4).cpu().numpy().astype(np.float64)
    t0 = t[t > 0].min()
    t = np.where(t > 0, (t - t0) / 1e3, np.nan)  # us from the first stamp
    ntiles = np.sum(~np.isnan(t[:, :, 0]), axis=1)
    mma = t[:, :, 1] - t[:, :, 0]
    epi_wait = t[:, :, 2] - t[:, :, 1]
    epi = t[:, :, 3] - t[:, :, 2]
    gap = t[:, 1:, 0] - t[:, :-1, 1]
    end = np.nanmax(t[:, :, 3], axis=1)
    print(f"{kind} M={M} N={N} K={K}: tiles/CTA {ntiles.min()}-{ntiles.max()}, first MMA start median "
          f"{np.nanmedian(t[:, 0, 0]):.2f} us, CTA end median {np.nanmedian(end):.2f} max {np.nanmax(end):.2f} us")
    print(f"   per tile: MMA issue span median {np.nanmedian(mma):.2f} us, acc->epilogue {np.nanmedian(epi_wait):.2f}, "
          f"epilogue {np.nanmedian(epi):.2f}, MMA gap between tiles {np.nanmedian(gap):.2f} us")
    c = int(np.nanargmax(end))
    print("   slowest CTA", c, ":", " | ".join(
        f"t{i}: mma {t[c, i, 0]:.1f}-{t[c, i, 1]:.1f} epi {t[c, i, 2]:.1f}-{t[c, i, 3]:.1f}" for i in range(ntiles[c])))


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "gpt2s"
    D = configs.WORKLOADS[name].ref
    M, d, F = 8192, D.hidden, D.ffn
    ao = D.num_heads * D.head_dim
    s = None
    X = torch.randn(M, max(d, F, ao), device="cuda").to(torch.bfloat16)
    for kind, N, K in (("o resid", d, ao), ("gate/up swiglu", 2 * F, d), ("down resid", d, F)):
        W = (torch.randn(N, K, device="cuda") * K ** -0.5).to(torch.bfloat16)
        Xk = X[:, :K].contiguous()
        if "resid" in kind:
            out = torch.zeros(M, N, device="cuda")
            run(kind, N, K, M, lambda: lib.fp_k_gemm_f32_residual(p(W), N, K, p(Xk), M, p(out), s))
        else:
            out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
            run(kind, N, K, M, lambda: lib.fp_k_gemm_swiglu(p(W), N // 2, K, p(Xk), M, p(out), s))


if __name__ == "__main__":
    main()
