"""Build the sm_100a extension in-tree: paper_2602_03529_b200/libsemstream_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a (never plain -arch, which also
embeds compute_100 PTX) with -fmad=false: the codec kernels reproduce numpy's
separately rounded float64 arithmetic bit-for-bit, so no FMA contraction.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
BUILD = PKG.parent / "build" / "csrc"
LIB = PKG / "libsemstream_b200.so"

SOURCES = ["capi.cu", "tma_host.cu", "encode.cu", "select.cu", "packet.cu", "decode.cu",
           "upscale.cu", "residual.cu", "learned.cu", "metrics.cu", "learned_i8.cu"]

# the learned-tokenizer kernels are bf16/fp32 tensor-core math with no
# bit-exact contract: let them contract a*b+c into FMA
FMAD_OK = {"learned.cu"}

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
    "-I", str(INCLUDE),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the semstream_b200 CUDA extension cannot be built")


def _stale(obj: Path, src: Path) -> bool:
    if not obj.exists():
        return True
    deps = [src] + list(CSRC.glob("*.cuh")) + list(INCLUDE.glob("*.h"))
    return any(d.stat().st_mtime > obj.stat().st_mtime for d in deps)


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(parents=True, exist_ok=True)
    exe = nvcc()
    jobs = []
    for name in SOURCES:
        src = CSRC / name
        obj = BUILD / (name[:-3] + ".o")
        if force or _stale(obj, src):
            flags = [f for f in NVCC_FLAGS if not (name in FMAD_OK and f == "-fmad=false")]
            jobs.append([exe, *flags, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and (r.stdout or r.stderr):
            print(r.stdout, r.stderr, file=sys.stderr)

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        list(ex.map(run, jobs))
    objs = [str(BUILD / (n[:-3] + ".o")) for n in SOURCES]
    if force or jobs or not LIB.exists():
        tmp = LIB.with_suffix(".so.tmp")
        run([exe, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", str(tmp), *objs,
             "-Xcompiler", "-fPIC"])
        os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
