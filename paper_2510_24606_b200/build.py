"""In-tree build of libdhsa_b200.so (sm_100a) with nvcc.

``python -m paper_2510_24606_b200.build`` compiles every ``csrc/*.cu`` to an
object in ``build/`` (in parallel) and links the shared library next to this
file, where ``_lib.py`` loads it.  The objects are rebuilt only when a source
or header is newer.
"""

from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "dhsa_b200")
LIB = os.path.join(PKG, "libdhsa_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", f"-I{INCLUDE}", f"-I{CSRC}"]
# extra nvcc flags, e.g. DHSA_NVCC_EXTRA=-DDHSA_SELECT_STAMPS for the select's
# phase stamps read by tools/step_timeline.py (objects rebuild when it changes)
EXTRA = os.environ.get("DHSA_NVCC_EXTRA", "").split()
FLAGS += EXTRA


def _deps():
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(INCLUDE, "*.h"))


def _stale(target, sources):
    if not os.path.exists(target):
        return True
    stamp = target + ".flags"
    if not os.path.exists(stamp) or open(stamp).read() != " ".join(EXTRA):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src, verbose):
    obj = os.path.join(BUILD, os.path.basename(src) + ".o")
    if not _stale(obj, [src] + _deps()):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    with open(obj + ".flags", "w") as f:
        f.write(" ".join(EXTRA))
    return obj, r.stderr if verbose else ""


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), sources))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    if _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcuda"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        with open(LIB + ".flags", "w") as f:
            f.write(" ".join(EXTRA))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
