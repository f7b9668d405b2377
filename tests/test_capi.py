"""The C-ABI libraries load (no GPU needed) and export every symbol declared
in include/*.h; the oracle build exports exactly the fp_sched.h surface."""
import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared(header):
    text = (ROOT / "include" / header).read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(fp_[a-z0-9_]+)\s*\(", text))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True).stdout
    return {l.split()[-1] for l in out.splitlines() if " T " in l}


def test_product_exports_every_declared_symbol():
    from paper_2409_13221_b200 import _lib
    lib = _lib.PRODUCT_LIB
    assert lib.exists(), "build first: python -c 'import __graft_entry__ as g; g.build()'"
    want = declared("fp_sched.h") | declared("fp_engine.h")
    missing = want - exported(lib)
    assert not missing, missing
    _lib.load()  # dlopen without a GPU and bind every ctypes signature


def test_ctypes_table_matches_headers():
    from paper_2409_13221_b200 import _lib
    assert set(_lib.SCHED_SYMBOLS) | set(_lib.ENGINE_SYMBOLS) == declared("fp_sched.h") | declared("fp_engine.h")


def test_oracle_library_exports_sched_surface():
    ref = ROOT / "oracle" / "_ref" / "libfuseplan_ref.so"
    if not ref.exists():
        pytest.skip("oracle/_ref not built")
    want = declared("fp_sched.h") - {"fp_fused_trigger"}  # product-only extension
    assert not (want - exported(ref))
    ctypes.CDLL(str(ref))


def test_engine_without_gpu_fails_loudly():
    """No silent CPU fallback: creating an engine without a device is an error."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2409_13221_b200 import _lib
    from paper_2409_13221_b200.configs import WORKLOADS
    from paper_2409_13221_b200.engine import Engine
    with pytest.raises(_lib.FpError):
        Engine(WORKLOADS["toy"])
