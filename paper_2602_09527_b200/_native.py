"""ctypes binding of the C ABI in include/proxtomo_b200.h.

The product path is the in-tree sm_100a library ``_lib/libproxtomo_b200.so``.
There is no CPU fallback: every entry point raises if the library or a CUDA
device is missing.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import build as _build

PT_OK, PT_EINVAL, PT_ECUDA, PT_EUNSUPPORTED, PT_ENCCL = 0, -1, -2, -3, -4
PT_RED_DOUBLES = 1025
EST_CODES = {"full": 0, "sgd": 1, "saga": 2, "svrg": 3, "lsvrg": 4}
SESSION_KINDS = {"fista": 5}  # include/proxtomo_b200.h PT_EST_FISTA
PROF_NAMES = ("fwd_band", "fwd_reduce", "gather_step", "fgp_call", "snapshot", "other",
              "snap_fwd_band", "snap_fwd_reduce", "snap_gather")

_lock = threading.Lock()
_lib = None

c_i32, c_i64, c_f32, c_f64, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_float,
                                    ctypes.c_double, ctypes.c_void_p)


class GeometryDesc(ctypes.Structure):
    _fields_ = [("height", c_i32), ("width", c_i32), ("n_slices", c_i32),
                ("n_angles", c_i32), ("n_bins", c_i32),
                ("bin_spacing", c_f64), ("pixel_size", c_f64),
                ("host_angles", ctypes.POINTER(c_f64)),
                ("row_offset", c_i32), ("rows_total", c_i32)]


class StepEpilogue(ctypes.Structure):
    _fields_ = [("estimator", c_i32), ("theta", c_i32), ("n_scale", c_f32),
                ("gamma", c_f32), ("hcoef", c_f32), ("iteration", c_i64),
                ("x", c_vp), ("h", c_vp), ("aux0", c_vp), ("aux1", c_vp),
                ("x_out", c_vp), ("v_out", c_vp), ("xhat_out", c_vp), ("bad_iter", c_vp)]


class SolverDesc(ctypes.Structure):
    _fields_ = [("estimator", c_i32), ("n_subsets", c_i32), ("gamma", c_f64),
                ("skip_probability", c_f64), ("prox_kind", c_i32), ("tv_alpha", c_f64),
                ("tv_inner", c_i32), ("tv_warm_start", c_i32), ("tv_nonneg", c_i32)]


_SIGS = {
    "pt_last_error": (ctypes.c_char_p, []),
    "pt_version": (ctypes.c_char_p, []),
    "pt_launch_count": (c_i64, []),
    "pt_geometry_desc_size": (c_i64, []),
    "pt_plan_create": (ctypes.c_int, [ctypes.POINTER(GeometryDesc), ctypes.POINTER(c_vp)]),
    "pt_plan_destroy": (ctypes.c_int, [c_vp]),
    "pt_selection_create": (ctypes.c_int, [c_vp, ctypes.POINTER(c_i32), c_i32, ctypes.POINTER(c_vp)]),
    "pt_selection_size": (c_i32, [c_vp]),
    "pt_selection_nnz": (c_i64, [c_vp, c_vp]),
    "pt_forward": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "pt_adjoint": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_f32, c_i32, c_vp]),
    "pt_adjoint_step": (ctypes.c_int, [c_vp, c_vp, c_vp, ctypes.POINTER(StepEpilogue), c_vp]),
    "pt_step_epilogue_apply": (ctypes.c_int, [c_vp, c_vp, ctypes.POINTER(StepEpilogue), c_vp]),
    "pt_fgp_workspace_floats": (c_i64, [c_vp]),
    "pt_tv_prox": (ctypes.c_int, [c_vp, c_vp, c_f64, c_i32, c_i32, c_vp, c_vp, c_vp, c_vp,
                                  c_vp, c_vp, c_f32, c_i64, c_vp, c_vp, c_vp]),
    "pt_tv_prox_emulate_rows": (ctypes.c_int, [c_vp, c_i32, c_vp, c_f64, c_i32, c_i32, c_vp, c_vp,
                                               c_vp, c_vp]),
    "pt_dot": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pt_tv_value": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp]),
    "pt_diff_norms": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pt_operator_norm_sq": (ctypes.c_int, [c_vp, c_vp, c_i32, ctypes.POINTER(c_f64), c_vp]),
    "pt_session_create": (ctypes.c_int, [c_vp, ctypes.POINTER(SolverDesc), c_vp, c_vp,
                                         ctypes.POINTER(c_vp), c_vp]),
    "pt_session_workspace_bytes": (c_i64, [c_vp, ctypes.POINTER(SolverDesc)]),
    "pt_session_create_in": (ctypes.c_int, [c_vp, ctypes.POINTER(SolverDesc), c_vp, c_vp, c_vp,
                                            c_i64, ctypes.POINTER(c_vp), c_vp]),
    "pt_session_destroy": (ctypes.c_int, [c_vp]),
    "pt_session_init": (ctypes.c_int, [c_vp, c_vp]),
    "pt_session_run": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(c_i32),
                                      ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(ctypes.c_uint8),
                                      c_i64, c_vp]),
    "pt_session_run_marked": (ctypes.c_int, [c_vp, c_i32, ctypes.POINTER(c_i32),
                                             ctypes.POINTER(ctypes.c_uint8),
                                             ctypes.POINTER(ctypes.c_uint8), c_i64, c_i32,
                                             ctypes.POINTER(c_i32), ctypes.POINTER(c_vp), c_vp]),
    "pt_session_x": (c_vp, [c_vp]),
    "pt_session_h": (c_vp, [c_vp]),
    "pt_session_buffer": (c_vp, [c_vp, c_i32]),
    "pt_session_bad_iter": (c_vp, [c_vp]),
    "pt_session_set_profiling": (ctypes.c_int, [c_vp, c_i32]),
    "pt_session_profile": (ctypes.c_int, [c_vp, ctypes.POINTER(c_f64), ctypes.POINTER(c_i64)]),
    "pt_session_emulate_sectors": (ctypes.c_int, [c_vp, c_i32]),
    "pt_pdhg_dual_sino": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pt_pdhg_dual_tv": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i32, c_i32, c_i32, c_f64, c_f64, c_vp]),
    "pt_pdhg_primal": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32, c_i32,
                                      c_i32, c_i64, c_vp, c_vp]),
    "pt_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint8)]),
    "pt_session_attach_nccl": (ctypes.c_int, [c_vp, ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint8),
                                              c_i32, c_i32]),
    "pt_session_attach_nccl_zslab": (ctypes.c_int, [c_vp, ctypes.c_char_p,
                                                    ctypes.POINTER(ctypes.c_uint8), c_i32, c_i32,
                                                    c_i32, c_i32]),
    "pt_session_emulate_zslabs": (ctypes.c_int, [c_vp, c_i32]),
    "pt_nccl_comm_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_uint8), c_i32,
                                           c_i32, ctypes.POINTER(c_vp)]),
    "pt_nccl_comm_destroy": (ctypes.c_int, [c_vp]),
    "pt_session_attach_comm": (ctypes.c_int, [c_vp, c_vp]),
    "pt_session_attach_comm_zslab": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32]),
    "pt_session_attach_comm_rows": (ctypes.c_int, [c_vp, c_vp, c_i32, c_i32]),
    "pt_session_override_rank": (ctypes.c_int, [c_vp, c_i32, c_i32]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)


def library_path() -> str:
    """The in-tree library; PT_LIB_OVERRIDE (A/B timing of two builds only)."""
    return os.environ.get("PT_LIB_OVERRIDE") or _build.LIB


def load(build_if_missing: bool = True):
    """Load (and if needed build) the native library; no device needed."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise RuntimeError(f"native library missing: {path}")
            _build.build()
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.pt_geometry_desc_size() != ctypes.sizeof(GeometryDesc):
            raise RuntimeError("pt_geometry_desc layout mismatch between include/proxtomo_b200.h "
                               "and this binding")
        _lib = lib
        return lib


def lib():
    """The library, for compute calls: requires a CUDA device (no fallback)."""
    if not torch.cuda.is_available():
        raise RuntimeError("proxtomo_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return load()


def check(rc: int, what: str = "") -> None:
    if rc == PT_OK:
        return
    msg = (load().pt_last_error() or b"").decode(errors="replace")
    text = f"{what}: {msg}" if what else msg
    if rc == PT_EINVAL:
        raise ValueError(text)
    raise RuntimeError(text)


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda or t.dtype not in (torch.float32, torch.float64, torch.int64) \
            or not t.is_contiguous():
        raise ValueError("expected a contiguous CUDA tensor")
    return int(t.data_ptr())


def launch_count() -> int:
    return int(load().pt_launch_count())


class _DeviceArray:
    """__cuda_array_interface__ view of library-owned device memory."""

    def __init__(self, address: int, shape, typestr: str = "<f4"):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": typestr,
            "data": (int(address), False), "version": 3, "strides": None,
        }


def device_view(address: int, shape, dtype=torch.float32) -> torch.Tensor:
    typestr = {torch.float32: "<f4", torch.int64: "<i8"}[dtype]
    return torch.as_tensor(_DeviceArray(address, shape, typestr), device="cuda")
