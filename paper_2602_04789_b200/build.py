"""Build the in-tree C-ABI library _lib/liblfattn.so for sm_100a with nvcc.

    python -m paper_2602_04789_b200.build
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc", "lfattn.cu")
OUT = os.path.join(HERE, "_lib", "liblfattn.so")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    d = os.path.join(HERE, "csrc")
    hdr = os.path.join(os.path.dirname(HERE), "include", "lfattn.h")
    return [os.path.join(d, f) for f in os.listdir(d)] + [hdr]


STAMP = OUT + ".flags"  # the extra nvcc flags the library was built with


def up_to_date(extra) -> bool:
    if not os.path.exists(OUT):
        return False
    try:
        built_with = open(STAMP).read()
    except OSError:
        built_with = ""
    if built_with != " ".join(extra):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    extra = os.environ.get("LF_NVCC_FLAGS", "").split()  # e.g. -DLF_V7_TRACE (event trace builds)
    if not force and up_to_date(extra):
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    tmp = OUT + ".tmp"
    cmd = [nvcc(), *FLAGS, *extra, "-o", tmp, SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, OUT)
    with open(STAMP, "w") as f:
        f.write(" ".join(extra))
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
