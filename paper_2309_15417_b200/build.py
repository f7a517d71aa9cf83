"""Build libltsgpu.so (sm_100a) in-tree with nvcc.

    python -m paper_2309_15417_b200.build [--force] [--verbose]

The library is plain CUDA C++ with a C ABI (include/ltsgpu.h); there is no
Python extension module and no JIT.  `-fmad=false` keeps every product and
sum separately rounded, which the bit-exact parity with the numpy
reference requires; the places where the reference itself uses FMA
(OpenBLAS) call __fma_rn explicitly.
"""

from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libltsgpu.so")
SOURCES = ["rows.cu", "search.cu", "unpack.cu", "broad.cu", "contacts.cu", "tree.cu"]
HEADERS = ["common.cuh", "geom.cuh", "dist_staged.cuh", "dist_tile.cuh", "moving.cuh", "bound32.cuh", "quat.cuh", "lapack3.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
    "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O2",
    "-Xptxas", "-warn-spills",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; set NVCC")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(REPO, "include", "ltsgpu.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build_fastpack(force: bool = False) -> str:
    """The host packing helper (csrc/fastpack.c, CPython C API) -> in-tree
    _fastpack<EXT_SUFFIX>, built with the system C compiler."""
    import sysconfig

    src = os.path.join(CSRC, "fastpack.c")
    dst = os.path.join(PKG, "_fastpack" + sysconfig.get_config_var("EXT_SUFFIX"))
    if not force and os.path.exists(dst) and os.path.getmtime(dst) >= os.path.getmtime(src):
        return dst
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        raise RuntimeError("no C compiler for the packing helper")
    tmp = dst + ".tmp"
    import numpy

    subprocess.run([cc, "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"], "-I", numpy.get_include(),
                    src, "-o", tmp], check=True)
    os.replace(tmp, dst)
    return dst


def build(force: bool = False, verbose: bool = False, extra=(), out: str | None = None) -> str:
    lib = out or LIB
    if out is None:
        build_fastpack(force)
    if out is None and not force and not _stale():
        return LIB
    import tempfile

    nvcc = nvcc_path()
    tmp = lib + ".tmp"
    # objects go to a private temporary directory that is removed whatever
    # happens (a failed compile leaves nothing next to the sources)
    with tempfile.TemporaryDirectory(prefix="ltsg_build_") as objdir:
        objs = []
        for src in SOURCES:
            obj = os.path.join(objdir, src.replace(".cu", ".o"))
            cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(REPO, "include"), "-c",
                   os.path.join(CSRC, src), "-o", obj]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
                print(" ".join(cmd), flush=True)
            subprocess.run(cmd, check=True)
            objs.append(obj)
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
               *objs, "-o", tmp]
        try:
            subprocess.run(cmd, check=True)
            os.replace(tmp, lib)
        finally:
            if os.path.exists(tmp):
                os.remove(tmp)
    return lib


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--out", default=None, help="build a variant library to this path")
    ap.add_argument("-D", dest="defines", action="append", default=[], help="extra -D for nvcc")
    args = ap.parse_args(argv)
    print(build(force=args.force, verbose=args.verbose, extra=[f"-D{d}" for d in args.defines],
                out=args.out))
    return 0


if __name__ == "__main__":
    sys.exit(main())
