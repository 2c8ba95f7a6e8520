"""Reference-side binding: a drop-in projector for ``proxtomo``'s own loop.

The reference's seam for the hot path is a duck-typed projector
(pkg/src/proxtomo/projector.py:143-167: ``forward(image, subset=None)``,
``adjoint(sino, subset=None)``, ``shape``, ``geometry``, ``width``,
``height``, ``norm_sq(iterations, seed)``); the estimators and the loop take
any such object (pkg/tests/test_estimators.py:69-82).  ``B200Projector`` is
that object over the C ABI of include/proxtomo_b200.h, bound with ctypes from
the header's struct layout alone -- numpy float64 in and out like the
reference, the device buffers owned by torch -- so a maintainer can hand it to
``proxtomo.solvers.run`` unchanged (Option B).

This module deliberately does not import the rest of the package: it is
what a maintainer would copy next to pkg/src/proxtomo/projector.py.  The
layout of ``pt_geometry_desc`` is asserted against the library at load
(``pt_geometry_desc_size``).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_DEFAULT_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib",
                            "libproxtomo_b200.so")


class _GeometryDesc(ctypes.Structure):
    """include/proxtomo_b200.h ``pt_geometry_desc``."""
    _fields_ = [("height", ctypes.c_int32), ("width", ctypes.c_int32),
                ("n_slices", ctypes.c_int32), ("n_angles", ctypes.c_int32),
                ("n_bins", ctypes.c_int32), ("bin_spacing", ctypes.c_double),
                ("pixel_size", ctypes.c_double),
                ("host_angles", ctypes.POINTER(ctypes.c_double)),
                ("row_offset", ctypes.c_int32), ("rows_total", ctypes.c_int32)]


_vp = ctypes.c_void_p
_lib = None


def load_library(path: str | None = None):
    """dlopen the ABI library once; refuse a struct layout that differs from ours."""
    global _lib
    if _lib is not None:
        return _lib
    lib = ctypes.CDLL(path or os.environ.get("PROXTOMO_B200_LIB", _DEFAULT_LIB))
    lib.pt_last_error.restype = ctypes.c_char_p
    lib.pt_geometry_desc_size.restype = ctypes.c_int64
    lib.pt_plan_create.argtypes = [ctypes.POINTER(_GeometryDesc), ctypes.POINTER(_vp)]
    lib.pt_plan_destroy.argtypes = [_vp]
    lib.pt_selection_create.argtypes = [_vp, ctypes.POINTER(ctypes.c_int32), ctypes.c_int32,
                                        ctypes.POINTER(_vp)]
    lib.pt_forward.argtypes = [_vp] * 8
    lib.pt_adjoint.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_float, ctypes.c_int32, _vp]
    lib.pt_operator_norm_sq.argtypes = [_vp, _vp, ctypes.c_int32, ctypes.POINTER(ctypes.c_double),
                                        _vp]
    have = int(lib.pt_geometry_desc_size())
    if have != ctypes.sizeof(_GeometryDesc):
        raise RuntimeError(f"pt_geometry_desc is {have} bytes in the library, "
                           f"{ctypes.sizeof(_GeometryDesc)} in this binding")
    _lib = lib
    return lib


def _check(rc: int) -> None:
    """PT_EINVAL -> ValueError (the reference's convention), others RuntimeError."""
    if rc == 0:
        return
    msg = (_lib.pt_last_error() or b"").decode(errors="replace")
    if rc == -1:
        raise ValueError(msg)
    raise RuntimeError(msg)


class B200Projector:
    """Duck-types ``proxtomo.projector.Projector`` (projector.py:143-167).

    ``geometry`` is any object with ``angles``, ``n_angles``, ``n_bins``,
    ``bin_spacing`` and ``pixel_size`` (the reference's ``ParallelGeometry``).
    Results are float64 numpy arrays computed in float32 on the device
    (projections within relative L2 1e-5 of the reference's float64)."""

    def __init__(self, geometry, width: int, height: int, library: str | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("B200Projector needs a CUDA device (there is no CPU fallback)")
        self._lib = load_library(library)
        self.geometry = geometry
        self.width = int(width)
        self.height = int(height)
        if self.width < 1 or self.height < 1:
            raise ValueError("width and height must be positive")
        angles = [float(a) for a in geometry.angles]
        self._angles = (ctypes.c_double * len(angles))(*angles)
        desc = _GeometryDesc(self.height, self.width, 1, len(angles), int(geometry.n_bins),
                             float(geometry.bin_spacing), float(geometry.pixel_size),
                             ctypes.cast(self._angles, ctypes.POINTER(ctypes.c_double)), 0, 0)
        self._plan = _vp()
        _check(self._lib.pt_plan_create(ctypes.byref(desc), ctypes.byref(self._plan)))
        self._selections: dict = {}

    def __del__(self):
        plan = getattr(self, "_plan", None)
        if plan and _lib is not None:
            try:
                torch.cuda.synchronize()
                _lib.pt_plan_destroy(plan)
            except Exception:
                pass

    @property
    def shape(self) -> tuple[int, int]:
        return (self.height, self.width)

    def _selection(self, subset):
        key = None if subset is None else tuple(int(i) for i in subset)
        hit = self._selections.get(key)
        if hit is None:
            handle = _vp()
            if key is None:
                _check(self._lib.pt_selection_create(self._plan, None, -1, ctypes.byref(handle)))
                n = len(self._angles)
            else:
                idx = (ctypes.c_int32 * max(1, len(key)))(*key)
                _check(self._lib.pt_selection_create(self._plan, idx, len(key),
                                                     ctypes.byref(handle)))
                n = len(key)
            hit = self._selections[key] = (handle, n)
        return hit

    @staticmethod
    def _stream() -> int:
        return int(torch.cuda.current_stream().cuda_stream)

    def forward(self, image, subset=None) -> np.ndarray:
        """projector.py:114-126: (H, W) -> (len(subset) or A, B)."""
        arr = np.asarray(image)
        if arr.shape != self.shape:
            raise ValueError(f"image shape {arr.shape} does not match grid {self.shape}")
        sel, n = self._selection(subset)
        x = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).cuda()
        y = torch.empty((n, int(self.geometry.n_bins)), device="cuda", dtype=torch.float32)
        if n:
            _check(self._lib.pt_forward(self._plan, sel, x.data_ptr(), None, None, y.data_ptr(),
                                        None, self._stream()))
        return y.double().cpu().numpy()

    def adjoint(self, sino, subset=None) -> np.ndarray:
        """projector.py:129-140: (len(subset) or A, B) -> (H, W)."""
        sel, n = self._selection(subset)
        arr = np.asarray(sino)
        if arr.shape != (n, int(self.geometry.n_bins)):
            raise ValueError(f"sinogram shape {arr.shape} does not match "
                             f"({n}, {self.geometry.n_bins})")
        y = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float32)).cuda()
        x = torch.zeros(self.shape, device="cuda", dtype=torch.float32)
        if n:
            _check(self._lib.pt_adjoint(self._plan, sel, y.data_ptr(), x.data_ptr(), 1.0, 0,
                                        self._stream()))
        return x.double().cpu().numpy()

    def norm_sq(self, iterations: int = 100, seed: int = 0) -> float:
        """projector.py:170-197: the start vector drawn exactly as the reference."""
        if iterations < 1:
            raise ValueError("iterations must be >= 1")
        rng = np.random.default_rng(seed)
        v = rng.standard_normal(self.width * self.height)
        while not np.any(v):
            v = rng.standard_normal(self.width * self.height)
        dv = torch.from_numpy(v.astype(np.float32)).cuda()
        out = ctypes.c_double()
        _check(self._lib.pt_operator_norm_sq(self._plan, dv.data_ptr(), int(iterations),
                                             ctypes.byref(out), self._stream()))
        return float(out.value)
