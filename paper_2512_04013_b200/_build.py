"""Build libaugsched.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libaugsched.so")
SOURCES = ["sim.cu", "step.cu", "gen.cu", "api.cu"]
HEADERS = ["model.cuh", "sim.cuh", "step.cuh", "select.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-fmad=false",                      # no FMA contraction in device code (R3)
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-Xcompiler", "-fvisibility=hidden",
    "-Xptxas", "-v",
]


def _nvcc():
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "augsched.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra_flags=()) -> str:
    """Compile libaugsched.so (or, with `out`, a variant such as the
    AUGSCHED_DEBUG build at DEBUG_LIB)."""
    dst = out or LIB
    if not force and out is None and not stale():
        return LIB
    if out is not None and not force and os.path.exists(dst) and os.path.getmtime(dst) >= os.path.getmtime(LIB) \
            and not stale():
        return dst
    extra = os.environ.get("AUGSCHED_NVCC_EXTRA", "").split()  # tuning experiments only
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, *extra_flags, "-shared", "-I", os.path.join(ROOT, "include"),
           *[os.path.join(CSRC, s) for s in SOURCES], "-o", dst + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + r.stdout + r.stderr)
    if verbose:
        print(r.stderr)
    os.replace(dst + ".tmp", dst)
    return dst


DEBUG_LIB = os.path.join(PKG, "libaugsched_debug.so")


def build_debug(force: bool = False) -> str:
    """The AUGSCHED_DEBUG build: device checks of the SURVEY §8(c).4
    invariants (sum of grants <= B, ledger A + P <= cap, the limit inside
    its clamp) latch E_STATE.  Loaded by setting AUGSCHED_LIB to its path."""
    return build(force=force, out=DEBUG_LIB, extra_flags=("-DAUGSCHED_DEBUG",))


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(LIB)
