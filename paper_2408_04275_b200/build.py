"""Builds libdisttrain_b200.so in-tree for sm_100a with nvcc.

Flags: -fmad=false (no FMA contraction: bit-exact with the CPU reference,
SURVEY.md Appendix A.1), no --use_fast_math, -lineinfo for ncu source views.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libdisttrain_b200.so")
OBJ = os.path.join(ROOT, "build", "obj")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v" if os.environ.get("DTB_PTXAS_V") else "-O3",
    "-I" + os.path.join(ROOT, "include"), "-I" + CSRC,
    "--expt-relaxed-constexpr",
] + [f"-D{d}" for d in os.environ.get("DTB_DEFINES", "").split() if d]
if os.environ.get("DTB_DEFINES"):  # experiment builds stay out of the product path
    OBJ = OBJ + "_" + "_".join(os.environ["DTB_DEFINES"].split()).replace("=", "")
    OUT = os.path.join(OBJ, "libdisttrain_b200.so")
SOURCES = ["capi.cu", "k_cost.cu", "k_intra.cu", "k_sched.cu", "k_inter.cu", "k_inter2.cu", "k_inter3.cu", "k_orch.cu",
           "k_misc.cu", "k_exhaustive.cu", "k_ingest.cu", "k_peer.cu"]


def _stale(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(ROOT, "include", "disttrain_b200.h"))

    def compile_one(src):
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src.replace(".cu", ".o"))
        if force or _stale([s] + headers, o):
            cmd = [NVCC, *FLAGS, "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
            if verbose and r.stderr:
                sys.stderr.write(r.stderr)
        return o

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    if force or _stale(objs, OUT):
        cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs,
               "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
