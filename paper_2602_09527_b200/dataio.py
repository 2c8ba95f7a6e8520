"""On-disk exchange with the reference's tools (host side).

The reference stores an image or sinogram as a JSON metadata file plus a
sibling ``<metadata-file-name>.raw`` payload of row-major little-endian
float64 values (pkg/src/proxtomo/dataio.py:19-117); sinogram metadata carries
the scan geometry, with an explicit angle list only for non-uniform scans.
This module writes and reads that same layout, so sinograms produced here
round-trip with ``proxtomo reconstruct`` and vice versa.  Device tensors are
accepted and returned as float64 numpy arrays (I/O is not on the hot path).
"""

from __future__ import annotations

import json
import os

import numpy as np

from .geometry import ParallelGeometry

_SIG = "<f8"


def _host64(a) -> np.ndarray:
    if hasattr(a, "detach"):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class _Record:
    """One metadata + payload pair."""

    def __init__(self, path: str):
        self.path = path
        self.payload_name = os.path.basename(path) + ".raw"
        self.payload_path = os.path.join(os.path.dirname(os.path.abspath(path)),
                                         self.payload_name)

    def write(self, meta: dict, values: np.ndarray) -> None:
        values.astype(_SIG, copy=False).tofile(self.payload_path)
        meta = dict(meta, payload=self.payload_name)
        with open(self.path, "w", encoding="utf-8") as fh:
            fh.write(json.dumps(meta, sort_keys=True, indent=2) + "\n")

    def read(self, kind: str) -> tuple[dict, callable]:
        with open(self.path, "r", encoding="utf-8") as fh:
            text = fh.read()
        try:
            meta = json.loads(text)
        except json.JSONDecodeError as exc:
            raise ValueError(f"malformed metadata in {self.path}: {exc}") from exc
        if not isinstance(meta, dict) or meta.get("kind") != kind:
            raise ValueError(f"{self.path} is not a {kind} file")

        def values(count: int) -> np.ndarray:
            raw = os.path.join(os.path.dirname(os.path.abspath(self.path)), meta["payload"])
            flat = np.fromfile(raw, dtype=_SIG)
            if flat.size != count:
                raise ValueError(f"payload {meta['payload']} holds {flat.size} values, "
                                 f"expected {count}")
            return flat.astype(np.float64)

        return meta, values


def save_image(path: str, image) -> None:
    img = _host64(image)
    if img.ndim != 2:
        raise ValueError("image must be 2D")
    _Record(path).write({"kind": "image", "height": int(img.shape[0]),
                         "width": int(img.shape[1])}, img)


def load_image(path: str) -> np.ndarray:
    meta, values = _Record(path).read("image")
    try:
        h, w = int(meta["height"]), int(meta["width"])
    except KeyError as exc:
        raise ValueError(f"image metadata missing key {exc}") from exc
    return values(h * w).reshape(h, w)


def save_sinogram(path: str, values, geometry: ParallelGeometry) -> None:
    sino = _host64(values)
    if sino.shape != (geometry.n_angles, geometry.n_bins):
        raise ValueError(f"sinogram shape {sino.shape} does not match geometry "
                         f"({geometry.n_angles}, {geometry.n_bins})")
    meta = {"kind": "sinogram", "n_angles": geometry.n_angles, "n_bins": geometry.n_bins,
            "bin_spacing": geometry.bin_spacing, "pixel_size": geometry.pixel_size}
    if not geometry.is_uniform():
        meta["angles"] = [float(a) for a in geometry.angles]
    _Record(path).write(meta, sino)


def load_sinogram(path: str) -> tuple[np.ndarray, ParallelGeometry]:
    meta, values = _Record(path).read("sinogram")
    try:
        n_angles, n_bins = int(meta["n_angles"]), int(meta["n_bins"])
        ds, h = float(meta["bin_spacing"]), float(meta["pixel_size"])
    except KeyError as exc:
        raise ValueError(f"sinogram metadata missing key {exc}") from exc
    if "angles" in meta:
        if len(meta["angles"]) != n_angles:
            raise ValueError("angles list does not match n_angles")
        geometry = ParallelGeometry(tuple(meta["angles"]), n_bins, ds, h)
    else:
        geometry = ParallelGeometry.uniform(n_angles, n_bins, ds, h)
    return values(n_angles * n_bins).reshape(n_angles, n_bins), geometry
