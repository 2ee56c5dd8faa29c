"""Build the sm_100a CUDA library in-tree (``paper_2108_01731_b200/_lib/liblcc_b200.so``).

Plain ``nvcc`` (no torch extension machinery): the product is a C-ABI
shared library, ``include/lcc_b200.h``.  ``-fmad=false`` keeps the fp64 gain
arithmetic free of FMA contraction so it matches the oracle bit for bit.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
SO = os.path.join(OUT_DIR, "liblcc_b200.so")
SOURCES = ["best_moves.cu", "apply.cu", "contract.cu", "objective.cu", "gen.cu", "eval.cu", "driver.cu", "memory.cu", "build.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
                "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
                "-Wno-deprecated-declarations", "-ccbin", "/usr/bin/g++"]


def _needs(obj: str, deps: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, extra: list[str] | None = None,
          out_dir: str | None = None) -> str:
    """Compile + link.  ``extra`` / ``out_dir``: tuning builds (A/B variants
    selected at run time with LCC_LIB_PATH); the product is the default."""
    out_dir = out_dir or OUT_DIR
    so = os.path.join(out_dir, "liblcc_b200.so")
    os.makedirs(out_dir, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
    headers.append(os.path.join(HERE, "..", "include", "lcc_b200.h"))
    jobs = []
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(out_dir, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _needs(obj, [sp] + headers):
            jobs.append([NVCC, *FLAGS, *(extra or []), "-c", sp, "-o", obj])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        if verbose and (r.stdout or r.stderr):
            print(r.stdout + r.stderr, file=sys.stderr)
        return cmd

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if jobs or not os.path.exists(so):
        run([NVCC, *ARCH, "-shared", "-o", so, *objs, "-lcudart"])
    return so


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
