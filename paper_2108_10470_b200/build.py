"""Build the in-tree CUDA library for sm_100a.

    python -m paper_2108_10470_b200.build

Compiles every csrc/*.cu with nvcc into _lib/libbsim_b200.so (one shared
object, C ABI in include/batchsim_b200.h).  No JIT: the .so ships in-tree.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libbsim_b200.so")
# measurement variant: IEEE fp32 (no FAST_FP32 flags), loaded with BSIM_LIB_VARIANT=ieee
OUT_IEEE = os.path.join(HERE, "_lib", "libbsim_b200_ieee.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


# fp32 arithmetic mode of the physics step TUs: flush-to-zero and the
# MUFU-based approximate divide / square root (<= 2 ulp; atan2f's internal
# divide, norms, the sweep's friction / cone-clamp square roots).  Measured
# 7 % faster step; fp64 (the exact-parity path) is unaffected,
# the task layer (bsim_tasks.cu) uses the same mode so the fused env step
# (task tail inside the physics kernel) is bitwise the two-launch path.
FAST_FP32 = ["-ftz=true", "-prec-div=false", "-prec-sqrt=false"]
FAST_TUS = ("bsim_step.cu", "bsim_step_large.cu", "bsim_tasks.cu")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(ROOT, "include", "batchsim_b200.h")]


def up_to_date(out=OUT):
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force=False, verbose=False, ieee=False, variant=None):
    """variant: a dev experiment build, _lib/libbsim_b200_<variant>.so with
    BSIM_NVCC_EXTRA's flags (loaded with BSIM_LIB_VARIANT=<variant>)."""
    out = OUT_IEEE if ieee else OUT
    if variant:
        out = os.path.join(HERE, "_lib", f"libbsim_b200_{variant}.so")
    if not force and up_to_date(out):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    from concurrent.futures import ThreadPoolExecutor
    tag = "_ieee" if ieee else (f"_{variant}" if variant else "")

    def compile_one(src):
        obj = os.path.join(HERE, "_lib", os.path.basename(src)[:-3] + tag + ".o")
        extra = os.environ.get("BSIM_NVCC_EXTRA", "").split()   # dev experiments only
        fast = (["-DBSIM_IEEE_FP32"] if ieee else
                FAST_FP32 if os.path.basename(src) in FAST_TUS else [])
        cmd = ["nvcc", *NVCC_FLAGS, *fast, *extra, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj]
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs = []
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as pool:   # one nvcc per TU
        for src, obj, r in pool.map(compile_one, sources()):
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            objs.append(obj)
    cmd = ["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs, "-o", out]
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, ieee="--ieee" in sys.argv))
