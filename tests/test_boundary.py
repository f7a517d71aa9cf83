"""The C-ABI boundary on CPU: the library loads, exports every symbol the
header declares, and the ctypes structs match the header layout."""

import ctypes
import os
import re

import pytest

from paper_2309_15417_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "ltsgpu.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ltsg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding_surface():
    assert set(_declared()) == set(_lib.EXPORTED)


@pytest.mark.skipif(not os.path.exists(_lib.LIB_PATH), reason="library not built")
def test_library_exports_every_declared_symbol():
    h = ctypes.CDLL(_lib.LIB_PATH)
    for name in _declared():
        assert hasattr(h, name), name
    assert _lib.lib().ltsg_version() == 1


def _c_struct_sizes():
    """Offsets of the last field per struct from a tiny C program (gcc)."""
    import subprocess
    import tempfile

    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "ltsgpu.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(ltsg_scene), offsetof(ltsg_scene, max_children),
         sizeof(ltsg_result), offsetof(ltsg_result, rows_bound),
         sizeof(ltsg_broad_input), offsetof(ltsg_broad_input, growth),
         sizeof(ltsg_broad_output), offsetof(ltsg_broad_output, ms),
         sizeof(ltsg_solve_input), offsetof(ltsg_solve_input, max_iterations),
         sizeof(ltsg_solve_output), offsetof(ltsg_solve_output, ms),
         sizeof(ltsg_integrate_input), offsetof(ltsg_integrate_input, separate));
  return 0;
}
'''
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        exe = os.path.join(d, "t")
        open(c, "w").write(prog)
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        return [int(x) for x in subprocess.run([exe], capture_output=True, text=True,
                                               check=True).stdout.split()]


def test_ctypes_structs_match_the_header():
    s, s_last, r, r_last, bi, bi_last, bo, bo_last, si, si_last, so, so_last, ii, ii_last = _c_struct_sizes()
    assert ctypes.sizeof(_lib.Scene) == s
    assert _lib.Scene.max_children.offset == s_last
    assert ctypes.sizeof(_lib.Result) == r
    assert _lib.Result.rows_bound.offset == r_last
    assert ctypes.sizeof(_lib.BroadInput) == bi
    assert _lib.BroadInput.growth.offset == bi_last
    assert ctypes.sizeof(_lib.BroadOutput) == bo
    assert _lib.BroadOutput.ms.offset == bo_last
    assert ctypes.sizeof(_lib.SolveInput) == si and _lib.SolveInput.max_iterations.offset == si_last
    assert ctypes.sizeof(_lib.SolveOutput) == so and _lib.SolveOutput.ms.offset == so_last
    assert ctypes.sizeof(_lib.IntegrateInput) == ii and _lib.IntegrateInput.separate.offset == ii_last


def test_missing_device_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a device is present")
    from paper_2309_15417_b200 import kernels

    with pytest.raises(_lib.LtsgError):
        kernels.feature_distances([[[0.0] * 3] * 3], [[[1.0] * 3] * 3])
