"""Builds the in-tree C-ABI library ``libnirc_b200.so`` for sm_100a.

Every ``csrc/*.cu`` is compiled with nvcc for ``-gencode
arch=compute_100a,code=sm_100a`` (cross-compiles without a GPU) and linked
into one shared object next to this file, so it travels to the GPU box with
the repo snapshot.  Rebuilds only when a source or header is newer than the
library.  Files listed in ``_NO_FMA`` are compiled with ``-fmad=false``.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libnirc_b200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
         "-Xcompiler", "-fPIC", "-I", INCLUDE]
# fp64 path walks: FMA contraction is on (measured -3 % render time; path
# lengths stay identical on every golden scene); NIRC_RENDER_FMAD=0 compiles
# render.cu with the reference's separate multiply/add rounding instead
_NO_FMA = {"render.cu"} if os.environ.get("NIRC_RENDER_FMAD") == "0" else set()


def _nvcc():
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found; cannot build the sm_100a library")
    return p


def _sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    return [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(INCLUDE, f) for f in os.listdir(INCLUDE)] + [__file__]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in _deps())


def _compile(src, verbose):
    obj = os.path.join(OBJ, src[:-3] + ".o")
    cmd = [_nvcc(), *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    if src in _NO_FMA:
        cmd.insert(1, "-fmad=false")
    if os.environ.get("NIRC_TRACE_MINB"):  # tuning experiments only
        cmd.insert(1, "-DNIRC_TRACE_MINB=" + os.environ["NIRC_TRACE_MINB"])
    for d in os.environ.get("NIRC_NVCC_DEFS", "").split():  # tuning experiments only
        cmd.insert(1, d)
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force=False, verbose=False):
    """Compile and link; returns the library path."""
    if not force and not needs_build():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if verbose:
        for _, err in results:
            sys.stderr.write(err)
    tmp = LIB + ".tmp"
    cmd = [_nvcc(), *ARCH, "-shared", "-o", tmp, *[o for o, _ in results], "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
