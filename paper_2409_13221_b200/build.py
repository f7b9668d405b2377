"""Build the in-tree native library paper_2409_13221_b200/lib/libfuseplan_b200.so.

Sources: csrc/host/*.cpp (C++20 scheduler = decision clock, C ABI of
include/fp_sched.h), csrc/engine/*.cpp|*.cu (per-GPU engine, executor, C ABI
of include/fp_engine.h) and csrc/kernels/*.cu (sm_100a kernels). CUDA code is
compiled only for sm_100a (`-gencode arch=compute_100a,code=sm_100a`); there
is no other target and no CPU fallback. Incremental by mtime; objects go to
build/ (git-ignored), the shared object into the package's lib/ so it travels
with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
REPO = PKG.parent
CSRC = PKG / "csrc"
OBJ = REPO / "build" / "obj"
LIB = PKG / "lib" / "libfuseplan_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CXX = os.environ.get("CXX", "g++")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INC = [f"-I{REPO / 'include'}", f"-I{CSRC / 'kernels'}", f"-I{CSRC / 'engine'}", "-I/usr/local/cuda/include"]
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-function", "-DFUSEPLAN_B200_EXTENSIONS"]
NVFLAGS = ["-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", *ARCH,
           *os.environ.get("FUSEPLAN_NVCC_EXTRA", "").split()]  # e.g. -DFP_GEMM_EXP (experiment builds)


def _sources():
    out = []
    for sub in ("host", "engine", "kernels"):
        d = CSRC / sub
        if d.is_dir():
            out += sorted(p for p in d.iterdir() if p.suffix in (".cpp", ".cu"))
    return out


def _headers():
    hs = list((REPO / "include").rglob("*.h*"))
    for sub in ("host", "engine", "kernels"):
        d = CSRC / sub
        if d.is_dir():
            hs += [p for p in d.iterdir() if p.suffix in (".h", ".cuh", ".hpp")]
    return hs


def _compile(src: Path, obj: Path, hdr_mtime: float):
    if obj.exists() and obj.stat().st_mtime >= max(src.stat().st_mtime, hdr_mtime):
        return None
    obj.parent.mkdir(parents=True, exist_ok=True)
    if src.suffix == ".cu":
        cmd = [NVCC, *NVFLAGS, *INC, "-c", str(src), "-o", str(obj)]
    else:
        cmd = [CXX, *CXXFLAGS, *INC, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {src}\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return str(src)


def build(verbose: bool = True, jobs: int | None = None) -> Path:
    srcs = _sources()
    hdr_mtime = max((h.stat().st_mtime for h in _headers()), default=0.0)
    objs = [OBJ / (s.parent.name + "_" + s.name + ".o") for s in srcs]
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 4))
    with cf.ThreadPoolExecutor(jobs) as ex:
        futs = [ex.submit(_compile, s, o, hdr_mtime) for s, o in zip(srcs, objs)]
        for f in futs:
            done = f.result()
            if done and verbose:
                print(f"[build] compiled {Path(done).relative_to(REPO)}", file=sys.stderr)
    newest = max(o.stat().st_mtime for o in objs)
    if not LIB.exists() or LIB.stat().st_mtime < newest:
        LIB.parent.mkdir(parents=True, exist_ok=True)
        cmd = [NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-Xlinker", "-Bsymbolic", *map(str, objs),
               "-o", str(LIB), "-lcudart_static", "-ldl", "-lrt", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose:
            print(f"[build] linked {LIB.relative_to(REPO)}", file=sys.stderr)
    return LIB


if __name__ == "__main__":
    build()
