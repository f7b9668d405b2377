"""One persistent decode-chain launch (csrc/kernels/chain.cu) at gpt2s widths for ncu:

    ncu --set full -k regex:decode_chain -s 2 -c 1 python tools/chain_probe.py [M]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2409_13221_b200 import _lib  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 284
d, H, KVH, hd, F, L, PT, max_pos = 768, 12, 12, 64, 3072, 3, 64, 600
lib = _lib.load()
g = torch.Generator(device="cuda").manual_seed(1)
r = lambda *s, sc=1.0: (torch.rand(*s, device="cuda", generator=g) * 2 - 1).mul_(sc).to(torch.bfloat16)  # noqa: E731
ao, qw = H * hd, (H + 2 * KVH) * hd
Wo, Wgu, Wd, Wqkv = r(d, ao, sc=ao ** -0.5), r(2 * F, d, sc=d ** -0.5), r(d, F, sc=F ** -0.5), r(qw, d, sc=d ** -0.5)
attn = r(M, ao)
x = torch.randn(M, d, device="cuda", generator=g)
g1, g2 = torch.ones(d, device="cuda"), torch.ones(d, device="cuda")
h = torch.zeros(M, d, device="cuda", dtype=torch.bfloat16)
act = torch.zeros(M, F, device="cuda", dtype=torch.bfloat16)
parts = torch.zeros(8, M, d, device="cuda")
q = torch.zeros(M, H, hd, device="cuda", dtype=torch.bfloat16)
maxp = (max_pos + PT - 1) // PT
pool = torch.zeros(M * maxp + 1, L, KVH, 2, PT, hd, device="cuda", dtype=torch.bfloat16)
bt = (torch.arange(M * maxp, device="cuda", dtype=torch.int32) + 1).view(M, maxp).contiguous()
slot = torch.arange(M, device="cuda", dtype=torch.int32)
pos = torch.randint(0, max_pos, (M,), device="cuda", generator=g, dtype=torch.int32)
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(4):
    assert lib.fp_k_decode_chain(p(Wo), p(Wgu), p(Wd), p(Wqkv), p(attn), p(h), p(act), p(parts), p(x), p(g1), p(g2),
                                 p(q), p(pool), L, 0, p(bt), maxp, p(slot), p(pos), max_pos, 10000.0, M, d, H, KVH,
                                 hd, F, None) == 0
torch.cuda.synchronize()
print("ok", M)
