"""Multi-GPU fused schedule on real B200s (needs >= 2 GPUs; skipped otherwise).

torchrun launches tests/mgpu_worker.py on 2 ranks: the long-tail migration
(KV pages pulled over NVLink through CUDA IPC) must execute exactly the
decision clock's moves, and the gathered experience must be bit-identical to
a single-GPU stage-barrier run of the same batch.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _gpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.parametrize("world", [2])
@pytest.mark.parametrize("mode,mech", [("forced", "kv"), ("greedy", "kv"), ("forced", "recompute")])
def test_fused_migration_matches_single_gpu(tmp_path, world, mode, mech):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    out = tmp_path / "res.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000),
           str(ROOT / "tests" / "mgpu_worker.py"), str(out), mode, mech]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert not res["plan"]["no_op"]
    assert res["plan"]["mechanism"] == ("kv_transfer" if mech == "kv" else "recompute_prefill")
    assert res["moves_match"], res
    assert res["handoff_ok"] and res["handoff_peer_bytes"] > 0, res
    assert res["bcast"]["same"] and res["bcast"]["changed"], res["bcast"]
    if mech == "kv":
        # KV pages are moved verbatim: bit-identical to the single-GPU run
        assert res["identical"], res["diffs_vs_1gpu"]
    else:
        # recompute re-prefills prompt + generated prefix with the prefill
        # kernels (different fp32 rounding than decode): tokens exact, log-probs
        # within the engine tolerance
        assert res["diffs_vs_1gpu"]["tokens"] == 0
        assert max(res["max_abs"].values()) <= 0.15, res["max_abs"]
