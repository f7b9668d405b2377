"""Phase timeline of tcgen05 GEMM CTAs (globaltimer stamps): where does a GEMM spend its time?

    python tools/gemm_trace.py            # decode-shaped cases of every epilogue
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib  # noqa: E402

lib = _lib.load()
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
tr = torch.zeros(8 * 65536, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["entry", "setup", "first_full", "last_full", "acc_ready", "epi_done"]


def case(kind, M, N, K):
    W = torch.randn(N, K, device="cuda").to(torch.bfloat16) * 0.05
    X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    if kind == "bf16":
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        f = lambda: lib.fp_k_gemm_bf16(p(W), N, K, p(X), M, p(out), N, None)  # noqa: E731
    elif kind == "swiglu":
        out = torch.empty(M, N // 2, device="cuda", dtype=torch.bfloat16)
        f = lambda: lib.fp_k_gemm_swiglu(p(W), N // 2, K, p(X), M, p(out), None)  # noqa: E731
    elif kind == "f32":
        s = lib.fp_k_gemm_splits(N, K)
        out = torch.empty(s, M, N, device="cuda")
        f = lambda: lib.fp_k_gemm_f32(p(W), N, K, p(X), M, p(out), s, None)  # noqa: E731
    elif kind == "qkvrope":  # decode QKV + RoPE + KV append (gpt2s heads)
        H, KVH, hd, L, PT = 12, 12, 64, 12, 64
        pos = torch.randint(0, 1000, (M,), device="cuda", dtype=torch.int32)
        maxp = 18
        pool = torch.zeros(M * maxp + 1, L, KVH, 2, PT, hd, device="cuda", dtype=torch.bfloat16)
        bt = (torch.arange(M * maxp, device="cuda", dtype=torch.int32) + 1).view(M, maxp)
        slot = torch.arange(M, device="cuda", dtype=torch.int32)
        q = torch.empty(M, H, hd, device="cuda", dtype=torch.bfloat16)
        f = lambda: lib.fp_k_qkv_rope(p(W), K, p(X), M, H, KVH, hd, p(pos), 1152, 10000.0, p(pool), L, 3, p(bt), maxp,  # noqa
                                      p(slot), p(q), None)
    else:  # vocab sampling head: A = X rows, B = W (vocab)
        sid = torch.arange(M, device="cuda", dtype=torch.int32)
        stp = torch.zeros(M, device="cuda", dtype=torch.int32)
        tok = torch.empty(M, device="cuda", dtype=torch.int32)
        lp = torch.empty(M, device="cuda")
        mode = int(os.environ.get("FP_VOCAB_MODE", "2"))  # 0 forced, 1 greedy, 2 sample
        tgt = torch.zeros(M, device="cuda", dtype=torch.int32)
        f = lambda: lib.fp_k_vocab(p(X), M, K, p(W), N, mode, 1.0, p(tgt) if mode == 0 else None, p(sid), p(stp), 7,  # noqa
                                   p(tok), p(lp), None)
    for _ in range(3):
        flush.zero_()
        tr.zero_()
        torch.cuda.synchronize()
        lib.fp_k_gemm_trace(p(tr))
        f()
        torch.cuda.synchronize()
        lib.fp_k_gemm_trace(None)
    t = tr.view(-1, 8).cpu().numpy()
    t = t[t[:, 0] > 0][:, :6].astype(np.float64)
    rel = (t - t[:, 0].min()) / 1000.0
    per = rel - rel[:, :1]
    print(f"{kind:6s} M={M} N={N} K={K} ctas={len(t)}: span {rel[:, 5].max():.2f} us | per-CTA med: "
          f"setup {np.median(per[:, 1]):.2f} first {np.median(per[:, 2]):.2f} main "
          f"{np.median(per[:, 3] - per[:, 2]):.2f} acc {np.median(per[:, 4] - per[:, 3]):.2f} "
          f"epi {np.median(per[:, 5] - per[:, 4]):.2f} total {np.median(per[:, 5]):.2f}", flush=True)


cases = (("qkvrope", 50, 2304, 768), ("qkvrope", 284, 2304, 768), ("bf16", 284, 2304, 768),
         ("swiglu", 284, 6144, 768), ("f32", 284, 768, 768), ("f32", 284, 768, 3072),
         ("bf16", 8, 2304, 768), ("bf16", 128, 2304, 768), ("swiglu", 8, 6144, 768), ("swiglu", 128, 6144, 768),
         ("f32", 8, 768, 768), ("f32", 128, 768, 768), ("f32", 8, 768, 3072), ("f32", 128, 768, 3072),
         ("vocab", 8, 50257, 768), ("vocab", 128, 50257, 768), ("vocab", 350, 50257, 768),
         ("bf16", 4096, 6144, 768), ("bf16", 16384, 2304, 768))
only = os.environ.get("FP_TRACE_ONLY")  # e.g. "vocab": run just those cases
for kind, M, N, K in cases:
    if not only or kind == only:
        case(kind, M, N, K)
