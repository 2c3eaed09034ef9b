"""Build libembrace.so in-tree for sm_100a (nvcc; no JIT cache).

Sources: paper_2110_09132_b200/csrc/*.cu; header: include/embrace.h.  NCCL is
the copy torch ships (nvidia/nccl), linked with an rpath so the same library
is used in-process by torch and by us.
"""

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libembrace.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
              "-Xptxas", "-v", "-Werror", "all-warnings"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for base in spec.submodule_search_locations:
            cands.append(os.path.join(base, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h not found (expected the nvidia-nccl wheel torch ships)")


def _nvcc():
    n = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(n):
        raise RuntimeError("nvcc not found")
    return n


def _stale(lib, srcs):
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = srcs + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(ROOT, "include", "embrace.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(s) > t for s in deps)


def build(force=False, verbose=False):
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    extra = os.environ.get("EMB_NVCC_EXTRA", "").split()  # e.g. -DEMB_TRACE (kernel trace builds)
    stamp = LIB + ".flags"
    same_flags = os.path.exists(stamp) and open(stamp).read() == " ".join(extra)
    if not force and same_flags and not _stale(LIB, srcs):
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    inc, libdir = _nccl_dirs()
    nvcc = _nvcc()
    common = ARCH + NVCC_FLAGS + ["-I", os.path.join(ROOT, "include"), "-I", inc]
    common += extra

    def comp(src):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = [nvcc, "-c", src, "-o", obj] + common
        r = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(BUILD, os.path.basename(src) + ".log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(comp, srcs))
    tmp = LIB + ".tmp"
    cmd = [nvcc, "-shared", "-o", tmp] + ARCH + objs + ["-L", libdir, "-l:libnccl.so.2",
                                                        "-Xlinker", "-rpath=" + libdir]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed:\n" + r.stderr[-4000:])
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(" ".join(extra))
    if verbose:
        print("built", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
