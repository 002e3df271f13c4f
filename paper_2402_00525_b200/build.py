"""Build the in-tree CUDA library ``libstp_b200.so`` for sm_100a with nvcc.

No torch extension machinery: the product is a plain C-ABI shared library
(include/stp.h) loaded with ctypes, so it travels with the repo snapshot and
is what the tests, smoke() and bench.py load.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libstp_b200.so")
SOURCES = ["stp_api.cu", "stp_preprocess.cu", "stp_sort.cu", "stp_render.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--shared",
         "-Xptxas", "-v", "-Wno-deprecated-gpu-targets"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cu", ".cuh"))] + \
        [os.path.join(os.path.dirname(HERE), "include", "stp.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, extra=(), out: str | None = None) -> str:
    """Build LIB (or ``out``: an A/B variant, e.g. variants/libstp_<tag>.so,
    with extra -D knobs)."""
    lib = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    extra = list(extra) + os.environ.get("STP_NVCC_EXTRA", "").split()
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    cmd = [nvcc(), *ARCH, *FLAGS, *[e for e in extra if e], *[os.path.join(CSRC, s) for s in SOURCES], "-o", lib + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(CSRC, "ptxas.log" if out is None else "ptxas_variant.log")
    with open(log, "w") as f:
        f.write(r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libstp_b200.so")
    os.replace(lib + ".tmp", lib)
    os.utime(lib, None)
    if verbose:
        sys.stdout.write(r.stderr)
    return lib


if __name__ == "__main__":
    # build.py [--force] | build.py --variant TAG -DKNOB=1 ...
    if "--variant" in sys.argv:
        i = sys.argv.index("--variant")
        tag, knobs = sys.argv[i + 1], sys.argv[i + 2:]
        print(build(force=True, extra=knobs, out=os.path.join(HERE, "variants", f"libstp_{tag}.so")))
    else:
        build(force="--force" in sys.argv, verbose=True)
