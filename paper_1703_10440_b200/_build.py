"""In-tree build of libaqr_b200.so for sm_100a (``python -m paper_1703_10440_b200._build``)."""

import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
SOURCES = [os.path.join(HERE, "csrc", "aqr_b200.cu")]
DEPENDS = SOURCES + sorted(glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + [
    os.path.join(REPO, "include", "aqr_b200.h")]
OUT = os.path.join(HERE, "libaqr_b200.so")
# The experiments build: the same library with the A/B knobs read from the
# environment (-DAQR_EXPERIMENTS; the shipped OUT ignores them).  Loaded via
# AQR_LIB_PATH by tests/test_gpu_variants.py and the tools/ab_*.sh scripts.
OUT_EXP = os.path.join(HERE, "libaqr_b200_exp.so")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xcompiler", "-fvisibility=hidden",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(p) <= t for p in DEPENDS)


def build(force=False, verbose=False, out=None, defines=()):
    """Build OUT (or `out` with extra -D `defines`, for tools/ A/B variants)."""
    if out is None and not force and up_to_date():
        return OUT
    target = out or OUT
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(REPO, "include"),
           "-o", target + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(target + ".tmp", target)
    return target


def build_experiments(force=False, verbose=False):
    if not force and os.path.exists(OUT_EXP) and all(os.path.getmtime(p) <= os.path.getmtime(OUT_EXP)
                                                    for p in DEPENDS):
        return OUT_EXP
    return build(out=OUT_EXP, defines=("AQR_EXPERIMENTS",), verbose=verbose)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--experiments" in sys.argv:
        print(build_experiments(force="--force" in sys.argv, verbose="-v" in sys.argv))
