"""In-tree build of the native libraries (nvcc for sm_100a, no JIT cache).

  libpspmm.so           the product: csrc/*.cu, csrc/*.cpp  (C ABI: include/pspmm.h)
  libpspmm_cusparse.so  the cuSPARSE SpMM baseline used only by bench.py and
                        tests (C ABI: include/pspmm_baseline.h)

python -m paper_2605_15695_b200.build_ext [--force] [--verbose]
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
# object files live outside the tree (only the .so files are in-tree and travel)
OBJROOT = os.environ.get("PSPMM_OBJ_DIR", os.path.join("/tmp", "pspmm_build"))
BUILD = os.path.join(OBJROOT, "obj")
LIB = os.path.join(PKG, "libpspmm.so")
LIB_CUSPARSE = os.path.join(PKG, "libpspmm_cusparse.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
          "--expt-relaxed-constexpr"]


def _sources():
    prod = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    prod = [s for s in prod if not os.path.basename(s).startswith("baseline_")]
    base = sorted(glob.glob(os.path.join(CSRC, "baseline_*.cu")))
    return prod, base


def _deps():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def _stale(target, inputs):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(i) > t for i in inputs)


def _compile(src, verbose=False, defines=(), objdir=None):
    obj = os.path.join(objdir or BUILD, os.path.basename(src) + ".o")
    if not _stale(obj, [src] + _deps()):
        return obj
    cmd = [NVCC] + ARCH + COMMON + [f"-D{d}" for d in defines] + ["-c", src, "-o", obj]
    if verbose and src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose:
        sys.stderr.write(r.stderr)
    return obj


def _link(objs, out, extra=()):
    tmp = out + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + list(extra)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed for {out}:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, out)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    prod, base = _sources()
    if force:
        for o in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        prod_objs = list(ex.map(lambda s: _compile(s, verbose), prod))
        base_objs = list(ex.map(lambda s: _compile(s, verbose), base))
    if force or _stale(LIB, prod_objs):
        _link(prod_objs, LIB)
    if base_objs and (force or _stale(LIB_CUSPARSE, base_objs)):
        _link(base_objs, LIB_CUSPARSE, ["-lcusparse"])
    return LIB


def build_variant(name: str, defines) -> str:
    """Same sources with extra -D flags (e.g. a register budget) into
    paper_2605_15695_b200/variants/libpspmm_<name>.so (experiments only)."""
    objdir = os.path.join(OBJROOT, f"obj_{name}")
    os.makedirs(objdir, exist_ok=True)
    out_dir = os.path.join(PKG, "variants")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, f"libpspmm_{name}.so")
    prod, _ = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, False, defines, objdir), prod))
    if _stale(out, objs):
        _link(objs, out)
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="--verbose" in sys.argv)
    print(LIB)
