"""One LM-head launch (fp_k_vocab) for ncu / timing: python tools/vocab_profile.py M mode(0 forced,1 greedy,2 sample) [persistent 0|1]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
mode = int(sys.argv[2]) if len(sys.argv) > 2 else 0
import os  # noqa: E402
V, K = map(int, os.environ.get("VOCAB_VK", "50257,768").split(","))
lib = _lib.load()
if len(sys.argv) > 3:  # 0: one tile per CTA instead of the persistent kernel (M >= 1024)
    lib.fp_k_set_packed_persistent(int(sys.argv[3]))
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
W = (torch.randn(V, K, device="cuda") * 0.05).to(torch.bfloat16)
X = torch.randn(M, K, device="cuda").to(torch.bfloat16)
tgt = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
sid = torch.arange(M, device="cuda", dtype=torch.int32)
stp = torch.zeros(M, device="cuda", dtype=torch.int32)
tok = torch.empty(M, device="cuda", dtype=torch.int32)
lp = torch.empty(M, device="cuda")
for _ in range(3):
    lib.fp_k_vocab(p(X), M, K, p(W), V, mode, 1.0, p(tgt), p(sid), p(stp), 7, p(tok), p(lp), None)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    lib.fp_k_vocab(p(X), M, K, p(W), V, mode, 1.0, p(tgt), p(sid), p(stp), 7, p(tok), p(lp), None)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"vocab M={M} mode={mode}: {ms * 1e3:.1f} us/launch (incl. alloc + finalize), "
      f"{2 * M * V * K / ms / 1e9:.0f} TFLOP/s")
