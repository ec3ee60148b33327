"""ctypes binding of libfastatlas.so (include/fastatlas.h).

This is the only route from Python into the product: every reference
function on the per-frame path is computed by the CUDA library.  There is
no CPU fallback — importing works anywhere (so `build()` and the CPU test
suite can inspect the library), but any compute call raises
`NativeUnavailable` unless the sm_100a library is built and a B200 is
visible.

Device memory and streams come from PyTorch (plumbing only); the library
receives raw device pointers.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading
import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FASTATLAS_LIB") or os.path.join(_HERE, "libfastatlas.so")
CSRC = os.path.join(_HERE, "csrc")

FA_OK = 0
FA_VALUE_ERROR = 1
FA_PACK_FAILURE = 2
FA_NOTHING_VISIBLE = 3
FA_HEIGHT_OVERFLOW = 4
FA_DEGENERATE_CHART = 5
FA_CUDA_ERROR = -1
FA_INTERNAL_ERROR = -2

# every symbol declared by include/fastatlas.h
EXPORTS = (
    "fa_abi_version", "fa_last_error", "fa_create", "fa_destroy", "fa_set_mesh", "fa_project",
    "fa_depth_prepass", "fa_mark_visible", "fa_build_adjacency", "fa_connected_charts", "fa_merge_shared_vertices",
    "fa_chart_boxes", "fa_blinn_clamped_ndc", "fa_select_side_plane", "fa_chart_bbox",
    "fa_viewport_box", "fa_orient", "fa_orient_order", "fa_fold", "fa_push_up", "fa_pack_at_scale",
    "fa_pack", "fa_frame_launch", "fa_frame_finish", "fa_frame", "fa_frame_download", "fa_frame_download_visible", "fa_frame_download_compact", "fa_frame_download_packed", "fa_vertex_order", "fa_last_launch_count",
    "fa_stage_times", "fa_stage_name", "fa_frame_counters", "fa_sequential_scale_search", "fa_sequential_pack", "fa_superblock_pack",
)


class NativeUnavailable(RuntimeError):
    """The CUDA library or a CUDA device is missing (there is no fallback)."""


class FrameParams(ctypes.Structure):
    _fields_ = [
        ("width", ctypes.c_int), ("height", ctypes.c_int),
        ("omega", ctypes.c_int64), ("n_scales", ctypes.c_int64),
        ("min_dim", ctypes.c_int64), ("padding", ctypes.c_int64),
        ("prescale", ctypes.c_double),
        ("backface_cull", ctypes.c_int), ("uv_f64", ctypes.c_int),
        ("want_depth", ctypes.c_int), ("use_graph", ctypes.c_int), ("profile", ctypes.c_int),
        ("packer", ctypes.c_int), ("block_size", ctypes.c_int64),
    ]


# fa_frame_params.packer (include/fastatlas.h): the make_packer registry, cli.py:318-339
PACKER_CODES = {"fastatlas": 0, "sequential": 1, "superblock": 2}


class FrameResult(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int), ("n_visible", ctypes.c_int32), ("n_charts", ctypes.c_int32),
        ("scale_num", ctypes.c_int64), ("scale_den", ctypes.c_int64),
        ("screen_fragments", ctypes.c_int64), ("texels_allocated", ctypes.c_int64),
        ("stretch_l2", ctypes.c_double), ("stretch_linf", ctypes.c_double), ("stretch_count", ctypes.c_int64),
        ("depth", ctypes.c_void_p), ("flags", ctypes.c_void_p), ("visible", ctypes.c_void_p),
        ("chart_of_triangle", ctypes.c_void_p), ("vertex_to_chart", ctypes.c_void_p),
        ("roots", ctypes.c_void_p), ("ndc", ctypes.c_void_p), ("px", ctypes.c_void_p),
        ("target", ctypes.c_void_p), ("placements", ctypes.c_void_p), ("uv", ctypes.c_void_p),
        ("visible_chart", ctypes.c_void_p),
        ("n_visible_vertices", ctypes.c_int64), ("visible_vertices", ctypes.c_void_p), ("vertex_uv", ctypes.c_void_p),
    ]


def build(force: bool = False) -> str:
    """Compile libfastatlas.so for sm_100a (make in csrc/)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC], check=True)
    else:
        subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


_lib = None
_lib_lock = threading.Lock()


def load_library():
    """Load the shared library (no device needed).  Raises NativeUnavailable."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i64, ci, cd = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
        sig = {
            "fa_abi_version": ([], ci),
            "fa_last_error": ([], ctypes.c_char_p),
            "fa_create": ([ctypes.POINTER(vp), ci], ci),
            "fa_destroy": ([vp], None),
            "fa_set_mesh": ([vp, vp, i64, vp, i64], ci),
            "fa_project": ([vp, vp, vp, vp], ci),
            "fa_depth_prepass": ([vp, vp, ci, ci, ci, vp, vp], ci),
            "fa_mark_visible": ([vp, vp, vp, ci, ci, ci, vp, vp], ci),
            "fa_build_adjacency": ([vp, vp, vp], ci),
            "fa_connected_charts": ([vp, vp, vp, vp, vp], ci),
            "fa_merge_shared_vertices": ([vp, vp, vp, vp, vp], ci),
            "fa_chart_boxes": ([vp, vp, vp, ci, ci, cd, vp, vp, vp, vp, vp, vp], ci),
            "fa_blinn_clamped_ndc": ([vp, vp, i64, vp, vp], ci),
            "fa_select_side_plane": ([vp, vp, i64, vp, vp], ci),
            "fa_chart_bbox": ([vp, vp, vp, i64, vp, vp], ci),
            "fa_viewport_box": ([vp, vp, i64, ci, ci, vp, vp], ci),
            "fa_orient": ([vp, vp, vp, i64, vp, vp, vp, vp], ci),
            "fa_orient_order": ([vp, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp], ci),
            "fa_fold": ([vp, vp, i64, i64, vp, vp, vp, vp], ci),
            "fa_push_up": ([vp, vp, vp, vp, vp, i64, i64, vp, vp, vp], ci),
            "fa_pack_at_scale": ([vp, vp, vp, i64, i64, i64, i64, i64, i64, vp, vp, vp, vp], ci),
            "fa_pack": ([vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, vp, vp], ci),
            "fa_frame_launch": ([vp, vp, ctypes.POINTER(FrameParams), vp], ci),
            "fa_frame_finish": ([vp, ctypes.POINTER(FrameResult), vp], ci),
            "fa_frame": ([vp, vp, ctypes.POINTER(FrameParams), ctypes.POINTER(FrameResult), vp], ci),
            "fa_frame_download": ([vp, ctypes.POINTER(FrameResult), vp, vp, vp, vp, vp], ci),
            "fa_frame_download_visible": ([vp, ctypes.POINTER(FrameResult), vp, vp, vp, vp, vp], ci),
            "fa_frame_download_compact": ([vp, ctypes.POINTER(FrameResult), vp, vp, vp, vp, vp, vp], ci),
            "fa_frame_download_packed": ([vp, ctypes.POINTER(FrameResult), vp, vp, vp, vp, vp, vp, vp], ci),
            "fa_vertex_order": ([vp, vp, vp], ci),
            "fa_last_launch_count": ([vp], ci),
            "fa_stage_times": ([vp, ctypes.POINTER(ctypes.c_float), ci, vp], ci),
            "fa_stage_name": ([ci], ctypes.c_char_p),
            "fa_frame_counters": ([vp, vp, ci], ci),
            "fa_sequential_scale_search": ([vp, vp, vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, vp], ci),
            "fa_superblock_pack": ([vp, vp, vp, vp, vp, i64, i64, i64, ci, vp, vp, vp, vp], ci),
            "fa_sequential_pack": ([vp, vp, vp, i64, i64, vp, vp, vp, vp, vp], ci),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
        return L


def last_error() -> str:
    return load_library().fa_last_error().decode("utf-8", "replace")


# --------------------------------------------------------------------------
# status -> reference exception
# --------------------------------------------------------------------------

def raise_for_status(code: int, what: str = "") -> None:
    if code == FA_OK:
        return
    msg = last_error() or what
    if code == FA_VALUE_ERROR:
        raise ValueError(msg)
    if code == FA_PACK_FAILURE:
        from .packing import PackFailure
        raise PackFailure(msg)
    if code == FA_HEIGHT_OVERFLOW:
        from .packing import HeightOverflow
        raise HeightOverflow(msg)
    if code == FA_DEGENERATE_CHART:
        from .geometry import DegenerateChart
        raise DegenerateChart(msg)
    if code == FA_NOTHING_VISIBLE:
        from .cli import NothingVisible
        raise NothingVisible(msg)
    raise RuntimeError(f"fastatlas error {code}: {msg}")


# --------------------------------------------------------------------------
# device plumbing (torch)
# --------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def require_device():
    torch = _torch()
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device visible; the B200 atlas path has no CPU fallback")
    load_library()
    return torch


class DevArray:
    """`__cuda_array_interface__` view of a context-owned device buffer."""

    def __init__(self, ptr: int, shape, dtype):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape),
            "typestr": np.dtype(dtype).str,
            "data": (int(ptr), False),
            "version": 3,
        }


def device_view(ptr, shape, dtype, device):
    """Zero-copy torch tensor over a context-owned buffer (valid until the next frame)."""
    torch = _torch()
    n = 1
    for s in shape:
        n *= int(s)
    if n == 0 or not ptr:
        return torch.empty(tuple(shape), dtype=_TORCH_DTYPES[np.dtype(dtype).str](), device=device)
    return torch.as_tensor(DevArray(ptr, shape, dtype), device=device)


_TORCH_DTYPES = {
    "<f8": lambda: _torch().float64, "<f4": lambda: _torch().float32, "<i4": lambda: _torch().int32,
    "<i8": lambda: _torch().int64, "|u1": lambda: _torch().uint8,
}


class Context:
    """One fa_ctx per (thread, device); owns scratch and frame outputs."""

    def __init__(self, device: int = 0):
        torch = require_device()
        self.device = int(device)
        self.torch_device = torch.device("cuda", self.device)
        L = load_library()
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            raise_for_status(L.fa_create(ctypes.byref(h), self.device), "fa_create")
        self.h = h
        self.L = L
        self._mesh_key = None

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.L.fa_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def stream_ptr(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def set_mesh(self, pos_t, tris_t):
        """Bind a mesh (fa_set_mesh keeps a renumbered device copy).  Re-binding
        the same unmodified live tensors is free; a different mesh, a
        freed-and-reallocated one (same pointers, new contents) or an in-place
        update of the bound tensors (their torch version counter moved, e.g. a
        deforming mesh) is bound again."""
        key = (pos_t.data_ptr(), tris_t.data_ptr(), pos_t.shape[0], tris_t.shape[0], pos_t._version,
               tris_t._version)
        prev = self._mesh_key
        if prev is None or prev[0] != key or prev[1]() is not pos_t or prev[2]() is not tris_t:
            raise_for_status(self.L.fa_set_mesh(self.h, ctypes.c_void_p(pos_t.data_ptr()), pos_t.shape[0],
                                                ctypes.c_void_p(tris_t.data_ptr()), tris_t.shape[0]))
            self._mesh_key = (key, weakref.ref(pos_t), weakref.ref(tris_t))


_contexts: dict = {}
_ctx_lock = threading.Lock()


def default_context(device: int | None = None) -> Context:
    torch = require_device()
    if device is None:
        device = torch.cuda.current_device()
    key = (threading.get_ident(), int(device))
    with _ctx_lock:
        c = _contexts.get(key)
        if c is None:
            c = Context(device)
            _contexts[key] = c
        return c


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def vp_host(view_proj) -> np.ndarray:
    m = np.ascontiguousarray(np.asarray(view_proj, dtype=np.float64).reshape(4, 4))
    return m
