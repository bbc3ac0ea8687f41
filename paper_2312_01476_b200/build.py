"""Build libsjb200.so in-tree with nvcc for sm_100a.

The library is one translation unit (csrc/sjb_capi.cu includes the kernel
sources) exporting the C ABI declared in include/simjoin_b200.h.  cudart is
linked statically so the .so only depends on the driver; it shares the
device's primary context with torch.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "libsjb200.so")
CSRC = os.path.join(PKG_DIR, "csrc")
HEADER = os.path.join(REPO_DIR, "include", "simjoin_b200.h")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [HEADER])


def is_stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(s) > t for s in sources())


def _locked(fn):
    """Run fn under an exclusive lock file next to the library, so concurrent
    processes (one per GPU under torchrun) never build into the same file."""
    import fcntl
    with open(os.path.join(PKG_DIR, ".build.lock"), "w") as fh:
        fcntl.flock(fh, fcntl.LOCK_EX)
        try:
            return fn()
        finally:
            fcntl.flock(fh, fcntl.LOCK_UN)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not is_stale() and os.path.exists(pack_ext_path()):
        return LIB_PATH
    return _locked(lambda: _build(force, verbose))


def _build(force: bool, verbose: bool) -> str:
    build_pack(force)
    if not force and not is_stale():      # another process built it meanwhile
        return LIB_PATH
    extra = os.environ.get("SJB_NVCC_EXTRA", "").split()   # e.g. -DSJB_PROFILE=1
    tmp = f"{LIB_PATH}.tmp{os.getpid()}"
    cmd = [_nvcc(), *NVCC_FLAGS, *extra, "-o", tmp, os.path.join(CSRC, "sjb_capi.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


def pack_ext_path() -> str:
    import sysconfig
    return os.path.join(PKG_DIR, "_sjbpack" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_pack(force: bool = False) -> str:
    """The CPython token packer (csrc/sjb_pack.c) -> _sjbpack<EXT_SUFFIX>."""
    import sysconfig
    out = pack_ext_path()
    src = os.path.join(CSRC, "sjb_pack.c")
    if not force and os.path.exists(out) and os.path.getmtime(out) > os.path.getmtime(src):
        return out
    tmp = f"{out}.tmp{os.getpid()}"
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-pthread",
           "-I" + sysconfig.get_paths()["include"], src, "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    print(build_pack(force="--force" in sys.argv))
