"""Matrix-free Joseph projector on the GPU, behind the reference's API.

Drop-in for pkg/src/proxtomo/projector.py:
  * ``forward_project`` (:114-126), ``back_project`` (:129-140),
  * ``Projector`` (:143-167), ``operator_norm_sq`` (:170-197).
The reference materialises A as a float64 scipy CSR matrix per
(geometry, grid) (:64-102); here a native *plan* holds only per-angle
parameters and both directions are evaluated on the fly by sm_100a kernels
(csrc/projector.cu).  Plans are cached like the reference's ``_tables``
(lru_cache(maxsize=8), :100-102).  Arrays in and out are float32 CUDA
tensors; numpy / CPU inputs are copied to the device.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict

import numpy as np
import torch

from . import _native as N
from .geometry import ParallelGeometry


def as_device(a, dtype=torch.float32) -> torch.Tensor:
    """Contiguous float32 CUDA tensor view/copy of a torch tensor or array."""
    N.lib()  # fail loudly without a device / library
    if isinstance(a, torch.Tensor):
        t = a
    else:
        t = torch.as_tensor(np.asarray(a))
    return t.to(device="cuda", dtype=dtype).contiguous()


class Plan:
    """Native plan: geometry + grid (+ slice count) and cached selections."""

    def __init__(self, geometry: ParallelGeometry, width: int, height: int, n_slices: int = 1,
                 row_slab: tuple | None = None):
        lib = N.lib()
        self.geometry = geometry
        self.width, self.height, self.n_slices = int(width), int(height), int(n_slices)
        # (row_offset, rows_total): the grid is rows [row_offset, row_offset + height)
        # of a rows_total-row image (multi-GPU rows decomposition)
        self.row_slab = None if row_slab is None else (int(row_slab[0]), int(row_slab[1]))
        r0, rt = self.row_slab if self.row_slab else (0, 0)
        self._angles = (ctypes.c_double * geometry.n_angles)(*geometry.angles)
        desc = N.GeometryDesc(self.height, self.width, self.n_slices, geometry.n_angles,
                              geometry.n_bins, float(geometry.bin_spacing),
                              float(geometry.pixel_size),
                              ctypes.cast(self._angles, ctypes.POINTER(ctypes.c_double)), r0, rt)
        handle = ctypes.c_void_p()
        N.check(lib.pt_plan_create(ctypes.byref(desc), ctypes.byref(handle)), "plan")
        self.handle = handle
        self._sel: dict = {}
        self._lock = threading.Lock()
        self._fgp_work = None

    def __del__(self):
        try:
            if getattr(self, "handle", None) and N._lib is not None:
                N._lib.pt_plan_destroy(self.handle)
        except Exception:
            pass

    def selection(self, subset=None):
        """Native selection handle for a subset (None = all angles, in order)."""
        key = None if subset is None else tuple(int(i) for i in subset)
        with self._lock:
            h = self._sel.get(key)
            if h is None:
                h = ctypes.c_void_p()
                if key is None:
                    N.check(N.lib().pt_selection_create(self.handle, None, -1, ctypes.byref(h)))
                else:
                    arr = (ctypes.c_int32 * max(1, len(key)))(*key)
                    N.check(N.lib().pt_selection_create(self.handle, arr, len(key),
                                                        ctypes.byref(h)), "subset")
                self._sel[key] = h
            return h

    def nnz(self, subset=None) -> int:
        return int(N.lib().pt_selection_nnz(self.handle, self.selection(subset)))

    @property
    def image_shape(self):
        if self.n_slices > 1:
            return (self.n_slices, self.height, self.width)
        return (self.height, self.width)

    def sino_shape(self, n_rows: int):
        if self.n_slices > 1:
            return (n_rows, self.n_slices, self.geometry.n_bins)
        return (n_rows, self.geometry.n_bins)

    def fgp_work(self) -> torch.Tensor:
        if self._fgp_work is None:
            n = int(N.lib().pt_fgp_workspace_floats(self.handle))
            self._fgp_work = torch.empty(n, device="cuda", dtype=torch.float32)
        return self._fgp_work

    # -- raw operator calls on device tensors --
    def forward_into(self, x, y, subset=None, x2=None, data=None, sumsq=None, stream=None):
        N.check(N.lib().pt_forward(self.handle, self.selection(subset), N.ptr(x), N.ptr(x2),
                                   N.ptr(data), N.ptr(y), N.ptr(sumsq), N.stream_handle(stream)),
                "forward")

    def adjoint_into(self, y, out, subset=None, alpha=1.0, accumulate=False, stream=None):
        N.check(N.lib().pt_adjoint(self.handle, self.selection(subset), N.ptr(y), N.ptr(out),
                                   float(alpha), int(bool(accumulate)), N.stream_handle(stream)),
                "adjoint")


_plans: "OrderedDict[tuple, Plan]" = OrderedDict()
_plans_lock = threading.Lock()


def get_plan(geometry: ParallelGeometry, width: int, height: int, n_slices: int = 1,
             row_slab: tuple | None = None) -> Plan:
    """lru_cache(maxsize=8) over (geometry, grid), like projector.py:100-102;
    plans hold device tables, so the current CUDA device is part of the key."""
    device = torch.cuda.current_device() if torch.cuda.is_available() else -1
    row_slab = None if row_slab is None else (int(row_slab[0]), int(row_slab[1]))
    key = (geometry, int(width), int(height), int(n_slices), row_slab, device)
    with _plans_lock:
        plan = _plans.get(key)
        if plan is not None:
            _plans.move_to_end(key)
            return plan
    plan = Plan(geometry, width, height, n_slices, row_slab)
    with _plans_lock:
        _plans[key] = plan
        while len(_plans) > 8:
            _plans.popitem(last=False)
    return plan


def _check_subset(subset, n_angles):
    """projector.py:105-111."""
    if subset is None:
        return None
    subset = tuple(int(i) for i in subset)
    if any(i < 0 or i >= n_angles for i in subset):
        raise ValueError(f"angle index out of range [0, {n_angles})")
    return subset


def forward_project(image, geometry: ParallelGeometry, subset=None) -> torch.Tensor:
    """Line integrals along every ray (projector.py:114-126).

    image (H, W) -> (n_selected, n_bins); a (Z, H, W) slice stack gives
    (n_selected, Z, n_bins) (slice-stacked 3D geometry)."""
    x = as_device(image)
    if x.ndim not in (2, 3):
        raise ValueError(f"image must be 2D, got shape {tuple(x.shape)}")
    subset = _check_subset(subset, geometry.n_angles)
    z = 1 if x.ndim == 2 else x.shape[0]
    plan = get_plan(geometry, x.shape[-1], x.shape[-2], z)
    n_rows = geometry.n_angles if subset is None else len(subset)
    y = torch.empty(plan.sino_shape(n_rows), device="cuda", dtype=torch.float32)
    plan.forward_into(x, y, subset)
    return y


def back_project(sino, geometry: ParallelGeometry, shape, subset=None) -> torch.Tensor:
    """Exact adjoint of :func:`forward_project` onto a (height, width) grid
    (projector.py:129-140); a per-pixel gather on the GPU."""
    y = as_device(sino)
    subset = _check_subset(subset, geometry.n_angles)
    n_rows = geometry.n_angles if subset is None else len(subset)
    shape = tuple(int(s) for s in shape)
    z = shape[0] if len(shape) == 3 else 1
    want = (n_rows, geometry.n_bins) if z == 1 else (n_rows, z, geometry.n_bins)
    if tuple(y.shape) != want:
        raise ValueError(f"sinogram shape {tuple(y.shape)} does not match {want}")
    plan = get_plan(geometry, shape[-1], shape[-2], z)
    out = torch.empty(shape, device="cuda", dtype=torch.float32)
    plan.adjoint_into(y, out, subset)
    return out


class Projector:
    """Forward/adjoint pair bound to one geometry and image grid
    (projector.py:143-167).  ``n_slices > 1`` = slice-stacked 3D volume
    (rotation about z), images (Z, H, W), sinograms (A, Z, B)."""

    def __init__(self, geometry: ParallelGeometry, width: int, height: int, n_slices: int = 1,
                 row_slab: tuple | None = None):
        self.geometry = geometry
        self.width = int(width)
        self.height = int(height)
        self.n_slices = int(n_slices)
        # (row_offset, rows_total): this grid is rows [row_offset, row_offset +
        # height) of a rows_total-row image; forward gives the slab's partial
        # line integrals (they add up over the slabs), adjoint the slab's rows
        self.row_slab = None
        if row_slab is not None:
            r0, rt = int(row_slab[0]), int(row_slab[1])
            if self.n_slices != 1 or r0 < 0 or r0 + self.height > rt:
                raise ValueError("row slab outside the image (or not 2D)")
            self.row_slab = (r0, rt)

    @property
    def shape(self) -> tuple:
        if self.n_slices > 1:
            return (self.n_slices, self.height, self.width)
        return (self.height, self.width)

    @property
    def plan(self) -> Plan:
        return get_plan(self.geometry, self.width, self.height, self.n_slices, self.row_slab)

    def forward(self, image, subset=None) -> torch.Tensor:
        x = as_device(image)
        if tuple(x.shape) != self.shape:
            raise ValueError(f"image shape {tuple(x.shape)} does not match grid {self.shape}")
        if self.row_slab is None:
            return forward_project(x, self.geometry, subset)
        subset = _check_subset(subset, self.geometry.n_angles)
        plan = self.plan
        n_rows = self.geometry.n_angles if subset is None else len(subset)
        y = torch.empty(plan.sino_shape(n_rows), device="cuda", dtype=torch.float32)
        plan.forward_into(x, y, subset)
        return y

    def adjoint(self, sino, subset=None) -> torch.Tensor:
        if self.row_slab is None:
            return back_project(sino, self.geometry, self.shape, subset)
        y = as_device(sino)
        subset = _check_subset(subset, self.geometry.n_angles)
        n_rows = self.geometry.n_angles if subset is None else len(subset)
        if tuple(y.shape) != (n_rows, self.geometry.n_bins):
            raise ValueError(f"sinogram shape {tuple(y.shape)} does not match "
                             f"{(n_rows, self.geometry.n_bins)}")
        out = torch.empty(self.shape, device="cuda", dtype=torch.float32)
        self.plan.adjoint_into(y, out, subset)
        return out

    def norm_sq(self, iterations: int = 100, seed: int = 0) -> float:
        return operator_norm_sq(self.geometry, self.width, self.height,
                                iterations=iterations, seed=seed, n_slices=self.n_slices)

    def __reduce__(self):
        return (Projector, (self.geometry, self.width, self.height, self.n_slices, self.row_slab))


def operator_norm_sq(geometry: ParallelGeometry, width: int, height: int,
                     iterations: int = 100, seed: int = 0, n_slices: int = 1) -> float:
    """Rayleigh-quotient power method on A^T A (projector.py:170-197).

    The start vector is the reference's ``default_rng(seed).standard_normal``
    draw (host, float64 -> float32); the iterations run on the GPU with
    float64 dot products."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    n = width * height * n_slices
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(n)
    while not np.any(v):
        v = rng.standard_normal(n)
    plan = get_plan(geometry, width, height, n_slices)
    dv = as_device(v.astype(np.float32))
    out = ctypes.c_double()
    N.check(N.lib().pt_operator_norm_sq(plan.handle, N.ptr(dv), int(iterations),
                                        ctypes.byref(out), N.stream_handle()), "norm_sq")
    return float(out.value)
