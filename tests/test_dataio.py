"""The reference's on-disk format (JSON metadata + raw little-endian float64,
pkg/src/proxtomo/dataio.py:19-117): round trips, and cross-compatibility with
the reference's own reader/writer when the reference is importable."""

import sys

import numpy as np
import pytest

from conftest import REFERENCE_SRC, reference_available
from paper_2602_09527_b200 import dataio
from paper_2602_09527_b200.geometry import ParallelGeometry


def test_roundtrip(tmp_path):
    rng = np.random.default_rng(0)
    img = rng.standard_normal((7, 5))
    dataio.save_image(str(tmp_path / "img.json"), img)
    assert np.array_equal(dataio.load_image(str(tmp_path / "img.json")), img)
    for g in (ParallelGeometry.uniform(6, 9, 0.5, 2.0), ParallelGeometry((0.0, 0.3, 1.1), 4)):
        s = rng.standard_normal((g.n_angles, g.n_bins))
        dataio.save_sinogram(str(tmp_path / "s.json"), s, g)
        s2, g2 = dataio.load_sinogram(str(tmp_path / "s.json"))
        assert np.array_equal(s2, s) and g2 == g
    with pytest.raises(ValueError):
        dataio.load_image(str(tmp_path / "s.json"))
    with pytest.raises(ValueError):
        dataio.save_sinogram(str(tmp_path / "bad.json"), np.zeros((2, 2)), g)


@pytest.mark.skipif(not reference_available(), reason="reference not mounted")
def test_cross_compatible_with_reference(tmp_path):
    sys.path.insert(0, REFERENCE_SRC)
    from proxtomo import dataio as ref_io
    from proxtomo.geometry import ParallelGeometry as RefGeometry
    rng = np.random.default_rng(1)
    g = ParallelGeometry.uniform(5, 8)
    s = rng.standard_normal((5, 8))
    dataio.save_sinogram(str(tmp_path / "ours.json"), s, g)
    s_ref, g_ref = ref_io.load_sinogram(str(tmp_path / "ours.json"))
    assert np.array_equal(s_ref, s) and g_ref.angles == g.angles
    ref_io.save_sinogram(str(tmp_path / "theirs.json"), s, RefGeometry.uniform(5, 8))
    s2, g2 = dataio.load_sinogram(str(tmp_path / "theirs.json"))
    assert np.array_equal(s2, s) and g2 == g
    img = rng.standard_normal((4, 6))
    ref_io.save_image(str(tmp_path / "im.json"), img)
    assert np.array_equal(dataio.load_image(str(tmp_path / "im.json")), img)
