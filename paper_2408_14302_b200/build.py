"""Build libwavehop_b200.so in-tree with nvcc for sm_100a (B200).

``python -m paper_2408_14302_b200.build`` (also called by ``__graft_entry__.build``).
The shared library is the product: hand-written CUDA for sm_100a behind the C ABI in
``include/wavehop_b200.h``.  It is built in-tree so it travels to the GPU box.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libwavehop_b200.so")
DIAG_LIB = os.path.join(HERE, "libwavehop_b200_diag.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3", "-shared",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.h")) + \
        [os.path.join(os.path.dirname(HERE), "include", "wavehop_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, diag: bool = False, dev: bool = False) -> str:
    """Build the product library; ``diag`` builds libwavehop_b200_diag.so instead (-DWH_DIAG:
    role switches, wait counters and the unit timeline compiled into the kernel; loaded by
    _lib when WH_DIAG_LIB=1 -- tools only, never the product path)."""
    lib = DIAG_LIB if diag else LIB
    if not force and not needs_build(lib):
        return lib
    # one nvcc per translation unit, in parallel, then one link
    objdir = os.path.join(HERE, "csrc", "build_diag" if diag else "build")
    os.makedirs(objdir, exist_ok=True)
    # dev (experiments only; never the shipped library): -DWH_DEV_BUILD instantiates two phase counts of the engine
    # kernel instead of seven -- for quick experiments on the large-hop paths
    cflags = [f for f in FLAGS if f != "-shared"] + (["-DWH_DIAG"] if diag else []) + \
        (["-DWH_DEV_BUILD"] if dev else []) + os.environ.get("WH_NVCC_EXTRA", "").split()
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        procs.append((src, obj, subprocess.Popen([NVCC, *cflags, "-c", "-o", obj, src],
                                                 stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
    log = []
    for src, obj, pr in procs:
        out, err = pr.communicate()
        log.append(err)
        if pr.returncode != 0:
            sys.stderr.write(out + err)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(src)}")
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", lib, *[o for _, o, _ in procs]]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed linking libwavehop_b200.so")
    if verbose:
        sys.stderr.write("".join(log))
    with open(os.path.join(HERE, "csrc", "ptxas_diag.log" if diag else "ptxas.log"), "w") as f:
        f.write("".join(log))
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, diag="--diag" in sys.argv, dev="--dev" in sys.argv))
