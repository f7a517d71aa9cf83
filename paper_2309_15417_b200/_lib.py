"""ctypes binding of libltsgpu.so (include/ltsgpu.h).

The library is loaded from the package directory only; there is no
fallback.  If it is missing, or no CUDA device is visible, every entry
point raises -- the narrow phase has no CPU path.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LTSG_LIB") or os.path.join(_HERE, "libltsgpu.so")

LTSG_OK, LTSG_EINVAL, LTSG_ECUDA, LTSG_ECAPACITY, LTSG_ENOMEM = 0, 1, 2, 3, 4

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32
F64 = C.c_double


class Scene(C.Structure):
    _fields_ = [
        ("tris", P), ("tri_orig", P), ("n_tris", I64),
        ("body_state", P), ("body_levels", P), ("n_bodies", I32), ("n_problems", I32),
        ("pair_body", P), ("pair_problem", P), ("pair_group", P), ("n_pairs", I64),
        ("problem_dt", P), ("problem_tbase", P),
        ("widen", F64), ("exhaustive", I32), ("max_children", I32),
    ]


class TreeUpload(C.Structure):
    """ltsg_tree_upload: the compact tree image ltsg_unpack_trees expands."""
    _fields_ = [
        ("verts", P), ("vidx", P), ("coarse", P), ("eps", P), ("kids", P), ("table", P),
        ("n_trees", I32), ("pad", I32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("dt", P), ("first_contact", P), ("collision", P), ("fused_offset", P),
        ("capacity", I64),
        ("body_a", P), ("body_b", P), ("position", P), ("normal", P), ("depth", P), ("t", P),
        ("tri_a", P), ("tri_b", P), ("threshold", P), ("problem", P),
        ("raw_problem", P), ("raw_body_a", P), ("raw_body_b", P), ("raw_position", P),
        ("raw_normal", P), ("raw_depth", P), ("raw_t", P), ("raw_tri_a", P), ("raw_tri_b", P),
        ("raw_threshold", P),
        ("n_fused", I64), ("n_raw", I64), ("rows_screen", I64), ("rows_zoom", I64),
        ("rows_bisect", I64), ("rows_executed", I64), ("candidates", I64),
        ("generations", I32), ("launches", I32),
        ("ms_screen", F64), ("ms_refine", F64), ("ms_contacts", F64),
        ("rows_screen_exact", I64), ("ms_exact", F64), ("ms_expand", F64), ("rows_bound", I64),
    ]


class BroadInput(C.Structure):
    """ltsg_broad_input (include/ltsgpu.h)."""
    _fields_ = [("particle", P), ("statics", P), ("n_particles", I32), ("n_statics", I32),
                ("dt_max", F64), ("growth", F64)]


class BroadOutput(C.Structure):
    """ltsg_broad_output (include/ltsgpu.h)."""
    _fields_ = [("dts", P), ("edge", P), ("window", P), ("link", P), ("cap_edges", I64), ("cap_links", I64),
                ("n_edges", I64), ("n_links", I64), ("candidates", I64), ("launches", I32), ("pad", I32),
                ("ms", F64)]


class SolveInput(C.Structure):
    """ltsg_solve_input (include/ltsgpu.h)."""
    _fields_ = [("body", P), ("n_bodies", I32), ("n_problems", I32), ("contact_offset", P), ("side", P),
                ("position", P), ("normal", P), ("t", P), ("n_contacts", I64), ("restitution", F64),
                ("friction", F64), ("relaxation", F64), ("penalty", F64), ("threshold", F64),
                ("max_iterations", I32), ("pad", I32)]


class SolveOutput(C.Structure):
    """ltsg_solve_output (include/ltsgpu.h)."""
    _fields_ = [("velocity", P), ("angular_velocity", P), ("touched", P), ("normal_impulse", P),
                ("friction_impulse", P), ("color", P), ("iterations", P), ("converged", P), ("launches", I32),
                ("pad", I32), ("ms", F64)]


class IntegrateInput(C.Structure):
    """ltsg_integrate_input (include/ltsgpu.h)."""
    _fields_ = [("body", P), ("n_bodies", I32), ("n_problems", I32), ("member_offset", P), ("member", P),
                ("t_new", P), ("contact_offset", P), ("side", P), ("id", P), ("normal", P), ("t", P), ("depth", P),
                ("n_contacts", I64), ("velocity", P), ("angular_velocity", P), ("touched", P), ("beta", F64),
                ("new_state_in", P), ("separate", I32), ("pad", I32)]


class TreeBuild(C.Structure):
    """ltsg_tree_build (include/ltsgpu.h)."""
    _fields_ = [("rec", P), ("eps", P), ("kids", P), ("steps", P), ("level_steps", P), ("level_keys", P),
                ("level_groups", P), ("n_levels", I32), ("fanout", I32), ("launches", I32), ("pad", I32)]


_lock = threading.Lock()
_lib = None


class LtsgError(RuntimeError):
    pass


class CapacityError(LtsgError):
    pass


class DeviceMemoryError(LtsgError):
    """cudaMalloc failed inside the workspace budget (LTSG_ENOMEM): a real
    out-of-memory, which splitting the batch would not cure."""


def lib():
    """The loaded library (loads on first use; raises if unavailable)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise LtsgError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2309_15417_b200.build` "
                "(the narrow phase has no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        h.ltsg_last_error.restype = C.c_char_p
        h.ltsg_version.restype = C.c_int
        for name, args in {
            "ltsg_point_triangle_closest": [P, P, P, P, I64, P, P, P],
            "ltsg_segment_segment_closest": [P, P, P, P, I64, P, P, P, P],
            "ltsg_feature_distances": [P, P, I64, P, P],
            "ltsg_closest_feature": [P, P, I64, P, P, P, P],
            "ltsg_overlap_centroid": [P, P, P, I64, P, P, P],
            "ltsg_search": [C.POINTER(Scene), C.POINTER(Result), P, P],
            "ltsg_exhaustive_rows": [C.POINTER(Scene), C.POINTER(I64), C.POINTER(I64), C.POINTER(F64), P, P],
            "ltsg_exhaustive_distances": [C.POINTER(Scene), P, C.POINTER(I64), P, P],
            "ltsg_fuse_contacts": [C.POINTER(Result), I64, P, P, P],
            "ltsg_fp64_peak": [C.POINTER(F64), C.POINTER(F64), P],
            "ltsg_unpack_trees": [C.POINTER(TreeUpload), P, P],
            "ltsg_broadphase": [C.POINTER(BroadInput), C.POINTER(BroadOutput), P, P],
            "ltsg_tube_rows": [P, P, P, P, P, P, P, P, P, I64, P, P, P],
            "ltsg_solve_impulses": [C.POINTER(SolveInput), C.POINTER(SolveOutput), P, P],
            "ltsg_integrate": [C.POINTER(IntegrateInput), P, P, P],
            "ltsg_build_trees": [C.POINTER(TreeBuild), P, P],
        }.items():
            fn = getattr(h, name)
            fn.argtypes = args
            fn.restype = C.c_int
        h.ltsg_workspace_create.argtypes = [I64]
        h.ltsg_workspace_create.restype = P
        h.ltsg_workspace_destroy.argtypes = [P]
        h.ltsg_workspace_destroy.restype = None
        h.ltsg_workspace_bytes.argtypes = [P]
        h.ltsg_workspace_bytes.restype = I64
        _lib = h
        return h


EXPORTED = (
    "ltsg_last_error", "ltsg_version", "ltsg_point_triangle_closest",
    "ltsg_segment_segment_closest", "ltsg_feature_distances", "ltsg_closest_feature",
    "ltsg_overlap_centroid", "ltsg_workspace_create", "ltsg_workspace_destroy",
    "ltsg_workspace_bytes", "ltsg_search", "ltsg_exhaustive_rows", "ltsg_exhaustive_distances", "ltsg_fuse_contacts", "ltsg_fp64_peak",
    "ltsg_unpack_trees", "ltsg_broadphase", "ltsg_tube_rows", "ltsg_solve_impulses", "ltsg_integrate",
    "ltsg_build_trees",
)


def check(rc: int, what: str) -> None:
    if rc == LTSG_OK:
        return
    msg = lib().ltsg_last_error().decode(errors="replace")
    if rc == LTSG_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if rc == LTSG_ECAPACITY:
        raise CapacityError(f"{what}: {msg}")
    if rc == LTSG_ENOMEM:
        raise DeviceMemoryError(f"{what}: {msg}")
    raise LtsgError(f"{what} failed ({rc}): {msg}")


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise LtsgError("no CUDA device visible: the B200 narrow phase has no CPU fallback")
    lib()
    return torch


class Workspace:
    """Owns an ltsg_workspace for one device; one per thread/stream."""

    def __init__(self, budget_bytes: int = 0):
        self.handle = lib().ltsg_workspace_create(int(budget_bytes))
        if not self.handle:
            raise LtsgError("ltsg_workspace_create failed")

    @property
    def nbytes(self) -> int:
        return int(lib().ltsg_workspace_bytes(self.handle))

    def close(self):
        if self.handle:
            lib().ltsg_workspace_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_tls = threading.local()


def workspace() -> Workspace:
    """Per-thread default workspace (the reference path is re-entrant and
    may be called from an engine thread pool, engine.py:183-193)."""
    import torch

    dev = torch.cuda.current_device()
    ws = getattr(_tls, "ws", None)
    if ws is None or getattr(_tls, "dev", None) != dev:
        ws = Workspace()
        _tls.ws = ws
        _tls.dev = dev
    return ws
