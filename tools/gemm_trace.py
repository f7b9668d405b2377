"""Phase timeline of tcgen05 GEMM CTAs (globaltimer stamps): where does a decode GEMM spend its time?"""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib  # noqa: E402

lib = _lib.load()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
tr = torch.zeros(8 * 8192, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["entry", "setup", "first_full", "last_full", "acc_ready", "epi_done"]
for M, N, K in ((16, 2304, 768), (256, 2304, 768), (64, 6144, 768), (350, 768, 3072), (4096, 6144, 768)):
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for rep in range(3):
        flush.zero_()
        tr.zero_()
        torch.cuda.synchronize()
        lib.fp_k_gemm_trace(p(tr))
        lib.fp_k_gemm_bf16(p(W), N, K, p(X), M, p(out), N, None)
        torch.cuda.synchronize()
        lib.fp_k_gemm_trace(None)
    t = tr.view(-1, 8).cpu().numpy()
    t = t[t[:, 0] > 0][:, :6].astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1000.0
    print(f"M={M} N={N} K={K} ctas={len(t)}: span {rel[:, 5].max():.2f} us")
    for i, nm in enumerate(names):
        print(f"   {nm:11s} min {rel[:, i].min():7.2f}  med {np.median(rel[:, i]):7.2f}  max {rel[:, i].max():7.2f}")
    d = rel[:, 3] - rel[:, 2]
    print(f"   mainloop(first->last full) med {np.median(d):.2f}  epi med {np.median(rel[:, 5] - rel[:, 4]):.2f}")
