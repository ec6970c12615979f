"""Build libhata.so in-tree with nvcc for sm_100a (no JIT, no torch types).

python -m paper_2506_02572_b200.build [-j N] [--force]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
INCLUDE = os.path.join(ROOT, "include")
# HATA_TRACE_BUILD=1: the diagnostics variant (phase stamps compiled in) for
# tools/trace_decode.py -> libhata_trace.so; the product is libhata.so
TRACE = os.environ.get("HATA_TRACE_BUILD") == "1"
# HATA_VARIANT=name HATA_DEFS="-DX=1 ...": an experimental build libhata_<name>.so
# (selected at run time with HATA_LIB); never the product
VARIANT = os.environ.get("HATA_VARIANT", "")
DEFS = os.environ.get("HATA_DEFS", "").split() if VARIANT else []
_name = "libhata" + ("_trace" if TRACE else "") + ("_" + VARIANT if VARIANT else "")
OUT = os.path.join(HERE, _name + ".so")
OBJ = os.path.join(HERE, "_build" + ("_trace" if TRACE else "") + ("_" + VARIANT if VARIANT else ""))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", INCLUDE, "-I", CSRC] + (["-DHATA_TRACE_ENABLED=1"] if TRACE else []) + DEFS
SOURCES = ["hata_abi.cu", "hata_decode.cu", "hata_hash.cu", "hata_hash_tc.cu", "hata_hash_umma.cu", "hata_shard.cu"]


def _deps():
    files = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(INCLUDE, "hata.h")]
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str) -> str:
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    log = obj + ".log"
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    return obj


def build(force: bool = False, jobs: int | None = None) -> str:
    if not force and os.path.exists(OUT) and os.path.getmtime(OUT) >= _deps():
        return OUT
    os.makedirs(OBJ, exist_ok=True)
    jobs = jobs or min(len(SOURCES), os.cpu_count() or 4)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = OUT + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    print(build(force=a.force, jobs=a.j))
    sys.exit(0)
