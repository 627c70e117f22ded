"""ctypes binding of libsbr200.so (include/sbr200.h).

The product path has no CPU fallback: if the CUDA library is missing or no
GPU is visible, every call raises ``NativeUnavailable``.  Build the library
with ``python -m paper_2604_09243_b200._build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes
import os
import threading
import weakref

import numpy as np

from .errors import NumericalError, SbrError, ValidationError

_PKG = os.path.dirname(os.path.abspath(__file__))
# SBR_LIB points at an alternative build (e.g. an instrumented variant)
LIB_PATH = os.environ.get("SBR_LIB") or os.path.join(_PKG, "libsbr200.so")

SBR_OK, SBR_EINVAL, SBR_EIO, SBR_ENUMERIC, SBR_ENOTSUP, SBR_ECUDA, SBR_ENCCL, SBR_ENOMEM = \
    0, 2, 3, 4, 5, 10, 11, 12
STORAGE_AUTO, STORAGE_F32_EXACT, STORAGE_F64, STORAGE_SINGLE = 0, 1, 2, 3
SEGMENT_RAYS = 1 << 19
TRAVERSAL_FAST, TRAVERSAL_REFERENCE = 0, 1


class NativeUnavailable(SbrError, RuntimeError):
    """The CUDA library could not be loaded or no device is usable."""


class CudaError(SbrError, RuntimeError):
    """A CUDA runtime failure inside the library."""


class CommError(SbrError, RuntimeError):
    """NCCL is unavailable or a collective failed (SBR_ENCCL)."""


c_i32, c_i64, c_dbl, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_double, ctypes.c_void_p


class Grid(ctypes.Structure):
    _fields_ = [("corner", c_dbl * 3), ("u", c_dbl * 3), ("v", c_dbl * 3),
                ("k", c_dbl * 3), ("spacing", c_dbl), ("cell_area", c_dbl),
                ("n_u", c_i64), ("n_v", c_i64)]


class TraceParams(ctypes.Structure):
    _fields_ = [("max_bounces", c_i32), ("strict", c_i32),
                ("allow_aliasing", c_i32), ("reserved", c_i32), ("eps", c_dbl),
                ("lambda_min", c_dbl), ("sampling_factor", c_dbl)]


SPLIT_MEDIAN, SPLIT_SAH, SPLIT_LBVH = 0, 1, 2


class BuildParams(ctypes.Structure):
    _fields_ = [("split_rule", c_i32), ("n_leaf", c_i32), ("max_depth", c_i32),
                ("bins_per_axis", c_i32), ("c_t", c_dbl), ("c_i", c_dbl)]


class Diag(ctypes.Structure):
    _fields_ = [("valid_rays", c_vp), ("max_bounce", c_vp), ("hist", c_vp),
                ("queries", c_vp)]


_SIGS = {
    "sbr_last_error": (ctypes.c_char_p, []),
    "sbr_abi_version": (ctypes.c_int, []),
    "sbr_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(c_vp)]),
    "sbr_ctx_destroy": (ctypes.c_int, [c_vp]),
    "sbr_ctx_synchronize": (ctypes.c_int, [c_vp]),
    "sbr_ctx_trim": (ctypes.c_int, [c_vp]),
    "sbr_ctx_stream": (ctypes.c_int, [c_vp, ctypes.POINTER(c_vp)]),
    "sbr_ctx_launch_count": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i64)]),
    "sbr_ctx_profile": (ctypes.c_int, [c_vp, c_i32]),
    "sbr_ctx_kernel_stats": (ctypes.c_int, [c_vp, ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64),
                                            ctypes.POINTER(c_dbl), ctypes.POINTER(c_i64)]),
    "sbr_ctx_raster_stats": (ctypes.c_int, [c_vp, ctypes.POINTER(c_dbl)]),
    "sbr_ctx_stage_ms": (ctypes.c_int, [c_vp, c_vp]),
    "sbr_ctx_raster_counters": (ctypes.c_int, [c_vp, c_vp]),
    "sbr_probe_l2_bandwidth": (ctypes.c_int, [c_vp, c_i64, c_i32, ctypes.POINTER(c_dbl)]),
    "sbr_ctx_debug_counters": (ctypes.c_int, [c_vp, c_vp, c_i32]),
    "sbr_debug_live_allocations": (ctypes.c_int, [ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "sbr_mesh_create": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32,
                                       ctypes.POINTER(c_vp)]),
    "sbr_mesh_destroy": (ctypes.c_int, [c_vp]),
    "sbr_mesh_info": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i32), c_vp]),
    "sbr_bvh_build": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(BuildParams),
                                     ctypes.POINTER(c_vp)]),
    "sbr_bvh_upload": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                                      ctypes.POINTER(c_vp)]),
    "sbr_bvh_info": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64),
                                    ctypes.POINTER(c_i32)]),
    "sbr_bvh_export": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sbr_bvh_destroy": (ctypes.c_int, [c_vp]),
    "sbr_closest_hit": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_dbl,
                                       c_vp, c_vp, c_vp]),
    "sbr_tri_hit_pairs": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl,
                                         c_dbl, c_i32, c_vp]),
    "sbr_aabb_hit_pairs": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_dbl, c_vp,
                                          c_vp]),
    "sbr_trace_grid": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(Grid),
                                      ctypes.POINTER(TraceParams), c_vp, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp]),
    "sbr_trace_grid_rows": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(Grid),
                                           ctypes.POINTER(TraceParams), c_i64, c_i64, c_vp,
                                           c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "sbr_trace_grid_hash": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(Grid),
                                           ctypes.POINTER(TraceParams), c_i64, c_i64, c_i64,
                                           c_vp]),
    "sbr_ctx_set_traversal": (ctypes.c_int, [c_vp, c_i32]),
    "sbr_packed_layout": (ctypes.c_int, [c_vp, c_i32, c_i32, c_i32, c_i32,
                                         ctypes.POINTER(c_i64)]),
    "sbr_solve_shard_packed": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32,
                                              ctypes.POINTER(TraceParams), c_vp, c_i32, c_dbl,
                                              c_i32, c_i32, c_i32, c_i32, c_vp]),
    "sbr_finalize_packed": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_i32, c_i32, c_i32, c_vp,
                                           c_vp, ctypes.POINTER(Diag)]),
    "sbr_comm_version": (ctypes.c_int, [ctypes.POINTER(c_i32)]),
    "sbr_comm_unique_id": (ctypes.c_int, [c_vp]),
    "sbr_comm_init": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp]),
    "sbr_comm_destroy": (ctypes.c_int, [c_vp]),
    "sbr_reduce_sum_f64": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i32]),
    "sbr_solve_distributed": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32,
                                             ctypes.POINTER(TraceParams), c_vp, c_i32, c_dbl,
                                             c_i32, c_i32, c_i32, c_vp, ctypes.POINTER(Diag)]),
    "sbr_ctx_get_traversal": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i32)]),
    "sbr_trace_rays": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64,
                                      ctypes.POINTER(TraceParams), c_vp, c_vp, c_vp, c_vp,
                                      c_vp, c_vp, c_vp]),
    "sbr_accumulate": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp,
                                      c_i32, c_dbl, c_dbl, c_i32, c_vp,
                                      ctypes.POINTER(c_i64)]),
    "sbr_solve": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32, ctypes.POINTER(TraceParams),
                                 c_vp, c_i32, c_dbl, c_i32, c_vp, ctypes.POINTER(Diag)]),
    "sbr_segment_layout": (ctypes.c_int, [c_vp, c_i32, c_vp]),
    "sbr_obj_read": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, ctypes.POINTER(c_vp)]),
    "sbr_obj_info": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "sbr_obj_copy": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "sbr_obj_free": (ctypes.c_int, [c_vp]),
    "sbr_obj_write": (ctypes.c_int, [ctypes.c_char_p, c_vp, c_vp, c_vp, c_i64]),
    "sbr_dump_hits_csv": (ctypes.c_int, [ctypes.c_char_p, c_i64, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "sbr_solve_shard": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i32,
                                       ctypes.POINTER(TraceParams), c_vp, c_i32, c_dbl, c_i32,
                                       c_i32, c_i32, c_i32, c_vp, c_vp]),
    "sbr_finalize": (ctypes.c_int, [c_vp, c_vp, c_i32, c_vp, c_i32, c_i32, c_vp, c_vp, c_vp,
                                    ctypes.POINTER(Diag)]),
}

EXPORTED = tuple(_SIGS)

_lib = None
_lib_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load libsbr200.so and bind every prototype (no GPU needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python -m paper_2604_09243_b200._build` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(rc: int, what: str = ""):
    if rc == SBR_OK:
        return
    msg = (_lib.sbr_last_error() or b"").decode("utf-8", "replace")
    text = f"{what}: {msg}" if what else msg
    if rc == SBR_EINVAL:
        raise ValidationError(msg)
    if rc == SBR_ENUMERIC:
        raise NumericalError(msg)
    if rc == SBR_EIO:
        raise OSError(text)
    if rc == SBR_ENOMEM:
        raise MemoryError(text)
    if rc == SBR_ENCCL:
        raise CommError(text)
    raise CudaError(f"[{rc}] {text}")


def obj_read(path):
    """Native OBJ parse (sbr_obj_read): (verts (V,3) f64, tris (T,3) i64,
    labels (T,) i64), or None when the file must be read by the Python loop
    (SBR_ENOTSUP: number syntax only Python defines; SBR_EIO: let Python's
    open() raise its own exception).  ValidationError as the reference."""
    import os
    lib = load_library()
    h = c_vp()
    rc = lib.sbr_obj_read(os.fsencode(path), str(path).encode("utf-8", "surrogateescape"),
                          ctypes.byref(h))
    if rc in (SBR_ENOTSUP, SBR_EIO):
        return None
    check(rc)
    try:
        nv, nt = c_i64(), c_i64()
        check(lib.sbr_obj_info(h, ctypes.byref(nv), ctypes.byref(nt)))
        verts = np.empty((nv.value, 3), np.float64)
        tris = np.empty((nt.value, 3), np.int64)
        labels = np.empty(nt.value, np.int64)
        check(lib.sbr_obj_copy(h, ptr(verts), ptr(tris), ptr(labels)))
    finally:
        lib.sbr_obj_free(h)
    return verts, tris, labels


def obj_write(path, v0, v1, v2) -> None:
    """Native save_obj (sbr_obj_write)."""
    import os
    lib = load_library()
    a = [f64(x, (-1, 3)) for x in (v0, v1, v2)]
    check(lib.sbr_obj_write(os.fsencode(path), *[ptr(x) for x in a], a[0].shape[0]),
          "sbr_obj_write")


def ptr(a) -> c_vp:
    if a is None:
        return c_vp(0)
    return c_vp(a.ctypes.data)


def f64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        out = out.reshape(shape)
    return out


# ---------------------------------------------------------------------------
# contexts: one per device, created lazily
# ---------------------------------------------------------------------------
class Context:
    def __init__(self, device: int):
        lib = load_library()
        h = c_vp()
        check(lib.sbr_ctx_create(int(device), ctypes.byref(h)), "sbr_ctx_create")
        self.handle = h
        self.device = int(device)
        self.lib = lib

    def synchronize(self):
        check(self.lib.sbr_ctx_synchronize(self.handle))

    def trim(self):
        """Return the grow-only solve/build scratch to the device (the next
        call re-grows it); meshes and trees stay resident."""
        check(self.lib.sbr_ctx_trim(self.handle), "sbr_ctx_trim")

    @property
    def launches(self) -> int:
        n = c_i64()
        check(self.lib.sbr_ctx_launch_count(self.handle, ctypes.byref(n)))
        return int(n.value)

    def profile(self, enable: bool = True):
        check(self.lib.sbr_ctx_profile(self.handle, int(bool(enable))))

    def kernel_stats(self) -> dict:
        tm, tn, pm, pn = c_dbl(), c_i64(), c_dbl(), c_i64()
        check(self.lib.sbr_ctx_kernel_stats(self.handle, ctypes.byref(tm), ctypes.byref(tn),
                                            ctypes.byref(pm), ctypes.byref(pn)))
        rm = c_dbl()
        check(self.lib.sbr_ctx_raster_stats(self.handle, ctypes.byref(rm)))
        ms = np.zeros(4)
        check(self.lib.sbr_ctx_stage_ms(self.handle, ptr(ms)))
        return {"trace_ms": tm.value, "trace_launches": int(tn.value), "po_ms": pm.value,
                "po_launches": int(pn.value), "raster_ms": float(ms[0]),
                "compact_ms": float(ms[1])}

    def raster_counters(self) -> dict:
        """Read and clear {candidates, wide_pairs, queue_overflows} of the
        raster pass (accumulated since the last read)."""
        out = np.zeros(3, np.int64)
        check(self.lib.sbr_ctx_raster_counters(self.handle, ptr(out)))
        return {"candidates": int(out[0]), "wide_pairs": int(out[1]),
                "queue_overflows": int(out[2])}

    @property
    def traversal(self) -> int:
        m = c_i32()
        check(self.lib.sbr_ctx_get_traversal(self.handle, ctypes.byref(m)))
        return int(m.value)

    @traversal.setter
    def traversal(self, mode: int):
        check(self.lib.sbr_ctx_set_traversal(self.handle, int(mode)), "sbr_ctx_set_traversal")

    @property
    def stream(self) -> int:
        s = c_vp()
        check(self.lib.sbr_ctx_stream(self.handle, ctypes.byref(s)))
        return int(s.value or 0)


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()


def live_allocations() -> tuple:
    """(count, bytes) of device allocations the library holds right now."""
    lib = load_library()
    n, b = c_i64(), c_i64()
    check(lib.sbr_debug_live_allocations(ctypes.byref(n), ctypes.byref(b)))
    return int(n.value), int(b.value)


# owning Python handles of device meshes / trees (geometry._DeviceMesh,
# bvh._DeviceBvh): shutdown() releases whatever is still alive
_handles: "weakref.WeakSet" = weakref.WeakSet()


def register_handle(obj) -> None:
    _handles.add(obj)


def shutdown() -> None:
    """Destroy every device object the library still holds -- trees, then
    meshes (any Python wrapper left alive is released and becomes unusable)
    -- and every device context with its scratch and streams.  Used by the
    leak check (scripts/sanitize_workload.py); afterwards
    live_allocations() is (0, 0)."""
    import gc
    gc.collect()
    live = list(_handles)
    for order in (0, 1):          # trees before the meshes they reference
        for h in live:
            if getattr(h, "is_tree", False) == (order == 0):
                h.release()
    with _ctx_lock:
        for dev, ctx in list(_contexts.items()):
            ctx.synchronize()
            check(ctx.lib.sbr_ctx_destroy(ctx.handle), "sbr_ctx_destroy")
            ctx.handle = None
            del _contexts[dev]


def current_device() -> int:
    env = os.environ.get("SBR_DEVICE")
    if env is not None:
        return int(env)
    try:
        import torch
        if torch.cuda.is_available():
            return int(torch.cuda.current_device())
    except Exception:  # pragma: no cover - torch is optional plumbing
        pass
    return 0


def context(device: int | None = None) -> Context:
    dev = current_device() if device is None else int(device)
    with _ctx_lock:
        ctx = _contexts.get(dev)
        if ctx is None:
            ctx = Context(dev)
            _contexts[dev] = ctx
        return ctx


def make_grid(grid) -> Grid:
    g = Grid()
    g.corner[:] = [float(x) for x in grid.corner]
    g.u[:] = [float(x) for x in grid.u]
    g.v[:] = [float(x) for x in grid.v]
    g.k[:] = [float(x) for x in grid.k_inc]
    g.spacing = float(grid.spacing)
    g.cell_area = float(grid.cell_area)
    g.n_u = int(grid.n_u)
    g.n_v = int(grid.n_v)
    return g


def make_trace_params(max_bounces, eps, strict=False, allow_aliasing=True,
                      lambda_min=0.0, sampling_factor=5.0) -> TraceParams:
    p = TraceParams()
    p.max_bounces = int(max_bounces)
    p.strict = int(bool(strict))
    p.allow_aliasing = int(bool(allow_aliasing))
    p.eps = float(eps)
    p.lambda_min = float(lambda_min)
    p.sampling_factor = float(sampling_factor)
    return p
