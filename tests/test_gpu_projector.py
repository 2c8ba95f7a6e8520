"""GPU parity of the matrix-free Joseph projector through the C ABI.

Tolerance (BASELINE.json north_star): projections within relative L2 1e-5 of
float64 -- the reference's own outputs (tests/golden) at desk sizes, the
pinned oracle at 512^2 / 2048^2 / 4096^2 subsets and for the 3D stack."""

import math

import numpy as np
import pytest
import torch

from conftest import rel_l2
from paper_2602_09527_b200 import (ParallelGeometry, Projector, back_project,
                                   build_staggered_partition, forward_project, operator_norm_sq)
from paper_2602_09527_b200 import _native as N

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _geom(units, ci):
    H, W, A, B, ds, h = units[f"p{ci}_meta"]
    return int(H), int(W), ParallelGeometry.uniform(int(A), int(B), float(ds), float(h))


def cpu(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("ci", range(8))
def test_projector_matches_reference_goldens(units, ci):
    H, W, g = _geom(units, ci)
    sub = tuple(int(i) for i in units[f"p{ci}_subset"])
    x = units[f"p{ci}_x"]
    if f"p{ci}_fwd" in units:
        assert rel_l2(cpu(forward_project(x, g)), units[f"p{ci}_fwd"]) <= TOL
        assert rel_l2(cpu(back_project(units[f"p{ci}_y"], g, (H, W))), units[f"p{ci}_adj"]) <= TOL
    assert rel_l2(cpu(forward_project(x, g, sub)), units[f"p{ci}_fwd_sub"]) <= TOL
    assert rel_l2(cpu(back_project(units[f"p{ci}_ys"], g, (H, W), sub)),
                  units[f"p{ci}_adj_sub"]) <= TOL


def test_selection_nnz_matches_reference_csr(units):
    for ci in range(8):
        H, W, g = _geom(units, ci)
        sub = tuple(int(i) for i in units[f"p{ci}_subset"])
        plan = Projector(g, W, H).plan
        assert plan.nnz(sub) == int(units[f"p{ci}_nnz_sub"])


@pytest.mark.parametrize("size,A,B,N", [(512, 720, 768, 20), (2048, 1800, 2900, 60)])
def test_projector_matches_oracle_at_config_sizes(oracle, size, A, B, N):
    """Configs 1 and 2: subsets 0 and N-1 against the float64 oracle (pinned to
    the reference at <= 1e-13); a smooth phantom plus noise."""
    from paper_2602_09527_b200 import problems
    g = ParallelGeometry.uniform(A, B)
    rng = np.random.default_rng(size)
    x = problems.ellipse_phantom(size, 20, 5) + 0.01 * rng.standard_normal((size, size))
    part = build_staggered_partition(A, N)
    oracle.set_mode("fast")
    try:
        for i in (0, N - 1):
            sub = part.subsets[i]
            y_ref = oracle.forward_project(x, g, sub)
            assert rel_l2(cpu(forward_project(x, g, sub)), y_ref) <= TOL
            r = rng.standard_normal(y_ref.shape)
            assert rel_l2(cpu(back_project(r, g, (size, size), sub)),
                          oracle.back_project(r, g, (size, size), sub)) <= TOL
    finally:
        oracle.set_mode("exact")


def test_projector_4096_subset_matches_oracle(oracle):
    """Config-4 projector size (4096^2, 3600 x 5800): a few angles incl. the
    diagonal and both branches."""
    A, B, n = 3600, 5800, 4096
    g = ParallelGeometry.uniform(A, B)
    sub = (0, 450, 900, 1350, 1801, 2700, 3599)
    rng = np.random.default_rng(4)
    from paper_2602_09527_b200 import problems
    x = problems.ellipse_phantom(n, 30, 9)
    oracle.set_mode("fast")
    try:
        y_ref = oracle.forward_project(x, g, sub)
        assert rel_l2(cpu(forward_project(x, g, sub)), y_ref) <= TOL
        r = rng.standard_normal(y_ref.shape)
        assert rel_l2(cpu(back_project(r, g, (n, n), sub)),
                      oracle.back_project(r, g, (n, n), sub)) <= TOL
    finally:
        oracle.set_mode("exact")


def test_adjoint_identity():
    g = ParallelGeometry.uniform(180, 192)
    rng = np.random.default_rng(0)
    for _ in range(5):
        x = rng.standard_normal((128, 128))
        y = rng.standard_normal((180, 192))
        lhs = float(np.sum(cpu(forward_project(x, g)) * y))
        rhs = float(np.sum(x * cpu(back_project(y, g, (128, 128)))))
        assert abs(lhs - rhs) <= 1e-5 * np.linalg.norm(x) * np.linalg.norm(y)


def test_zero_image_and_linearity():
    g = ParallelGeometry.uniform(7, 11)
    assert torch.count_nonzero(forward_project(np.zeros((9, 9)), g)) == 0
    rng = np.random.default_rng(2)
    g = ParallelGeometry.uniform(45, 71)
    x, z = rng.standard_normal((48, 48)), rng.standard_normal((48, 48))
    combo = cpu(forward_project(2.5 * x - 1.25 * z, g))
    parts = 2.5 * cpu(forward_project(x, g)) - 1.25 * cpu(forward_project(z, g))
    assert rel_l2(combo, parts) <= 1e-6


def test_subset_rows_concatenate_bitwise():
    """projector.py:86-97: A_S is a row slice of A -- the native kernel gives
    bitwise the same rows whichever selection they are computed in."""
    rng = np.random.default_rng(3)
    g = ParallelGeometry.uniform(90, 101)
    x = rng.standard_normal((64, 64))
    full = cpu(forward_project(x, g))
    for n in (2, 3, 7):
        rebuilt = np.empty_like(full)
        for sub in build_staggered_partition(90, n).subsets:
            rebuilt[list(sub)] = cpu(forward_project(x, g, sub))
        assert np.array_equal(rebuilt, full)


def test_central_pixel_chord_known_answer():
    """tests/test_projector.py:18-30 of the reference."""
    g = ParallelGeometry.uniform(8, 9)
    img = np.zeros((9, 9))
    img[4, 4] = 1.0
    sino = cpu(forward_project(img, g))
    for a, th in enumerate(g.angles):
        assert sino[a].argmax() == 4
        chord = 1.0 / max(abs(math.cos(th)), abs(math.sin(th)))
        assert sino[a, 4] == pytest.approx(chord, rel=1e-6)
        assert np.all(sino[a, :3] == 0.0) and np.all(sino[a, 6:] == 0.0)


def test_disc_analytic_chords():
    """tests/test_projector.py:33-49 of the reference (non-unit spacings)."""
    n, h, radius = 200, 2.0 / 200, 0.7
    g = ParallelGeometry.uniform(5, 61, bin_spacing=0.03, pixel_size=h)
    c = (np.arange(n) - (n - 1) / 2) * h
    yy, xx = np.meshgrid(c, c, indexing="ij")
    disc = ((xx ** 2 + yy ** 2) <= radius ** 2).astype(float)
    sino = cpu(forward_project(disc, g))
    s = (np.arange(61) - 30) * 0.03
    chord = 2.0 * np.sqrt(np.maximum(radius ** 2 - s ** 2, 0.0))
    err = np.abs(sino - chord[None, :])
    interior = np.abs(s) <= radius - 5 * h
    assert err[:, interior].max() <= 2.0 * h
    assert np.linalg.norm(err) / np.linalg.norm(chord) <= 0.02


def test_validation_errors():
    g = ParallelGeometry.uniform(5, 9)
    with pytest.raises(ValueError):
        forward_project(np.zeros((4, 4)), g, subset=(0, 5))
    with pytest.raises(ValueError):
        back_project(np.zeros((2, 9)), g, (4, 4), subset=(-1, 0))
    with pytest.raises(ValueError):
        back_project(np.zeros((4, 9)), g, (4, 4))
    with pytest.raises(ValueError):
        forward_project(np.zeros(16), g)


def test_operator_norm_matches_reference(units):
    g = ParallelGeometry.uniform(60, 95)
    assert operator_norm_sq(g, 64, 64, 50, 0) == pytest.approx(float(units["norm_desk"]), rel=1e-5)
    g = ParallelGeometry.uniform(10, 23)
    assert operator_norm_sq(g, 16, 16, 100, 0) == pytest.approx(float(units["norm_small"]), rel=1e-5)


def test_slice_stacked_3d_matches_per_slice_oracle(oracle):
    """Config-3 geometry: rotation about z, every slice an independent 2D
    problem (reference 2D operator per slice)."""
    g = ParallelGeometry.uniform(36, 48)
    rng = np.random.default_rng(7)
    vol = rng.standard_normal((5, 32, 32))
    sub = tuple(range(1, 36, 4))
    proj = Projector(g, 32, 32, n_slices=5)
    y = cpu(proj.forward(vol, sub))
    assert y.shape == (len(sub), 5, 48)
    for z in range(5):
        assert rel_l2(y[:, z], oracle.forward_project(vol[z], g, sub)) <= TOL
    r = rng.standard_normal((len(sub), 5, 48))
    xa = cpu(proj.adjoint(r, sub))
    for z in range(5):
        assert rel_l2(xa[z], oracle.back_project(r[:, z], g, (32, 32), sub)) <= TOL


def test_native_launch_counter_moves():
    before = N.launch_count()
    forward_project(np.ones((16, 16)), ParallelGeometry.uniform(4, 9))
    torch.cuda.synchronize()
    assert N.launch_count() > before


_TILE_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r})
import oracle as O
from paper_2602_09527_b200 import ParallelGeometry, back_project
g = ParallelGeometry.uniform(37, 301)
rng = np.random.default_rng(3)
y = rng.standard_normal((37, 301))
sub = tuple(range(0, 37, 2))
ys = y[list(sub)]
got = back_project(ys, g, (190, 211), sub).double().cpu().numpy()
O.set_mode("fast")
ref = O.back_project(ys, g, (190, 211), sub)
print(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
"""


@pytest.mark.parametrize("tile", [0, 1, 2, 3])
def test_every_gather_tile_matches_oracle(tile):
    """Each gather tile shape (the plan picks one by image size) against the oracle."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PT_GATHER_TILE=str(tile))
    out = subprocess.run([sys.executable, "-c", _TILE_SNIPPET.format(repo=repo)], env=env,
                         check=True, capture_output=True, text=True, timeout=300)
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-5


_FWD_CFG_SNIPPET = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r})
import oracle as O
from paper_2602_09527_b200 import ParallelGeometry, forward_project
g = ParallelGeometry.uniform(41, 771)
x = np.random.default_rng(5).random((530, 512))
sub = tuple(range(1, 41, 3))
got = forward_project(x, g, sub).double().cpu().numpy()
O.set_mode("fast")
ref = O.forward_project(x, g, sub)
print(float(np.linalg.norm(got - ref) / np.linalg.norm(ref)))
"""


@pytest.mark.parametrize("cfg,tma", [(c, "1") for c in range(8)] + [(3, "0"), (4, "0")])
def test_every_forward_tile_config_matches_oracle(cfg, tma):
    """Each forward band/tile configuration (PT_FWD_CFG, images from 512 up;
    the plan's default is 3), with row-branch tiles by TMA or by cp.async
    (PT_FWD_TMA=0), against the oracle on a non-square image with ragged bands
    and tiles."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PT_FWD_CFG=str(cfg), PT_FWD_TMA=tma)
    out = subprocess.run([sys.executable, "-c", _FWD_CFG_SNIPPET.format(repo=repo)], env=env,
                         check=True, capture_output=True, text=True, timeout=300)
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-5


@pytest.mark.parametrize("size,A,B", [(128, 180, 192), (64, 60, 95), (40, 36, 60)])
def test_small_forward_tma_and_cp_async_staging_agree_bitwise(oracle, size, A, B):
    """Images <= 128^2 take the one-launch forward: its image is staged by one
    TMA box when the image is 16-byte aligned with W % 4 == 0, else by cp.async
    into an odd-pitch buffer.  The staged values are the same, so an image at
    a 4-byte offset (cp.async) projects to the same bits as the aligned copy
    (TMA); both match the float64 oracle."""
    g = ParallelGeometry.uniform(A, B)
    rng = np.random.default_rng(size)
    x = rng.standard_normal((size, size))
    xa = torch.tensor(x, device="cuda", dtype=torch.float32)
    store = torch.empty(size * size + 1, device="cuda", dtype=torch.float32)
    xm = store[1:].view(size, size)  # 4 bytes past a 16-byte boundary
    xm.copy_(xa)
    assert xa.data_ptr() % 16 == 0 and xm.data_ptr() % 16 == 4
    sub = tuple(range(1, A, 7))
    for s in (sub, None):
        ya = forward_project(xa, g, s)
        ym = forward_project(xm, g, s)
        assert torch.equal(ya, ym)
        y_ref = oracle.forward_project(x, g, s)
        assert rel_l2(cpu(ya), y_ref) <= TOL


def test_random_small_geometries_match_oracle(oracle):
    """Seeded random small problems (both sides <= 128: the one-launch
    forward; odd and even widths: its TMA and cp.async staging; bin spacing
    and pixel size != 1: two-tap and multi-candidate gathers) against the
    float64 oracle, full and subset selections."""
    rng = np.random.default_rng(20261021)
    for _ in range(12):
        H, W = int(rng.integers(3, 129)), int(rng.integers(3, 129))
        A, B = int(rng.integers(1, 41)), int(rng.integers(3, 220))
        ds = float(rng.choice([0.5, 0.7, 1.0, 1.3]))
        h = float(rng.choice([0.8, 1.0, 1.5]))
        g = ParallelGeometry.uniform(A, B, ds, h)
        x = rng.standard_normal((H, W))
        sub = tuple(sorted(rng.choice(A, size=max(1, A // 3), replace=False).tolist()))
        for s in (None, sub):
            y_ref = oracle.forward_project(x, g, s)
            assert rel_l2(cpu(forward_project(x, g, s)), y_ref) <= TOL, (H, W, A, B, ds, h)
            r = rng.standard_normal(y_ref.shape)
            assert rel_l2(cpu(back_project(r, g, (H, W), s)),
                          oracle.back_project(r, g, (H, W), s)) <= TOL, (H, W, A, B, ds, h)
