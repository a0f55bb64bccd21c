"""In-tree build of the native libraries (no JIT cache, so the .so files
travel to the GPU box with the repo snapshot).

    python -m paper_2011_06391_b200.build          # build what is stale
    python -m paper_2011_06391_b200.build --force  # rebuild everything

Products (git-ignored, gpurun-shipped):
    paper_2011_06391_b200/lib/libfusedmm_cuda.so  sm_100a kernels + C ABI
    paper_2011_06391_b200/lib/libfmm_gen.so       host input generators
    oracle/_build/libfmm_oracle.so                CPU oracle (test infra)
    oracle/_ref/libfusedmm_ref.so                 reference, when present
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"
OBJ = PKG / "lib" / "obj"
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xptxas", "-warn-spills", f"-I{INCLUDE}", f"-I{CSRC}"]
if os.environ.get("FMM_TUNING") == "1":  # tuning variants of the row kernels (tests/sweep_variants.py)
    NVCC_FLAGS.append("-DFMM_TUNING_VARIANTS")
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-march=x86-64-v3", f"-I{INCLUDE}", f"-I{CSRC}"]

CUDA_SOURCES = ["fmm_api.cu", "fmm_k_sigmoid.cu", "fmm_k_gcn.cu", "fmm_k_fr.cu",
                "fmm_k_tdist.cu", "fmm_k_frattr.cu", "fmm_k_generic.cu", "fmm_k_stream.cu", "fmm_unfused.cu",
                "fmm_ingest.cu"]
HOST_SOURCES = ["fmm_plan.cpp", "fmm_mmio.cpp", "fmm_mt64.cpp"]


def _newest_dep() -> float:
    deps = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return max((p.stat().st_mtime for p in deps), default=0.0)


def _stale(out: Path, srcs: list[Path], dep_time: float) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(s.stat().st_mtime > t for s in srcs) or dep_time > t


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")


def build_cuda(force: bool = False, jobs: int | None = None) -> Path:
    if shutil.which(NVCC) is None and not Path(NVCC).exists():
        raise RuntimeError(f"nvcc not found at {NVCC}")
    OBJ.mkdir(parents=True, exist_ok=True)
    dep = _newest_dep()
    steps = []
    objs = []
    for s in CUDA_SOURCES:
        src = CSRC / s
        o = OBJ / (s + ".o")
        objs.append(o)
        if force or _stale(o, [src], dep):
            steps.append([NVCC, *NVCC_FLAGS, "-c", str(src), "-o", str(o)])
    for s in HOST_SOURCES:
        src = CSRC / s
        o = OBJ / (s + ".o")
        objs.append(o)
        if force or _stale(o, [src], dep):
            steps.append(["g++", *CXX_FLAGS, "-c", str(src), "-o", str(o)])
    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        list(ex.map(_run, steps))
    out = LIB / "libfusedmm_cuda.so"
    if force or steps or _stale(out, objs, 0.0):
        _run([NVCC, *ARCH, "-shared", "-o", str(out), *map(str, objs), "-cudart", "static"])
    return out


def build_gen(force: bool = False) -> Path:
    LIB.mkdir(parents=True, exist_ok=True)
    out = LIB / "libfmm_gen.so"
    src = CSRC / "fmm_gen.cpp"
    if force or _stale(out, [src], 0.0):
        _run(["g++", "-O3", "-std=c++17", "-fPIC", "-march=x86-64-v3", "-pthread", "-shared", "-o", str(out),
              str(src)])
    return out


def build_oracle(force: bool = False) -> None:
    """CPU checkers (oracle/Makefile). Building the checker is not using it."""
    cmd = ["make", "-s", "-C", str(ROOT / "oracle")]
    if force:
        subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), "clean"], check=False)
    _run(cmd)


def build_all(force: bool = False) -> None:
    build_gen(force)
    build_oracle(force)
    build_cuda(force)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--only", choices=["cuda", "gen", "oracle"], default=None)
    a = ap.parse_args()
    if a.only == "cuda":
        print(build_cuda(a.force))
    elif a.only == "gen":
        print(build_gen(a.force))
    elif a.only == "oracle":
        build_oracle(a.force)
    else:
        build_all(a.force)
        print("built:", LIB / "libfusedmm_cuda.so")
