"""GPU parity of the temporally blocked FGP TV prox (regularizers.py:90-133).

float32 on the device vs the reference's float64: tolerance 1e-4 relative L2
(the north_star's iterate tolerance); the blocked kernel is also checked
against an unblocked run of itself (T = 1 per launch is what the oracle
does) through many launch splits."""

import numpy as np
import pytest
import torch

from conftest import rel_l2
from paper_2602_09527_b200 import TvProxConfig, nonneg_prox, tv_prox, tv_value

pytestmark = pytest.mark.gpu


def cpu(t):
    return t.detach().double().cpu().numpy()


@pytest.mark.parametrize("nn", [0, 1])
def test_fgp_matches_reference_goldens(units, nn):
    u = units["fgp_u"]
    cfg = TvProxConfig(alpha=0.5, inner_iterations=37, nonneg=bool(nn))
    x, st = tv_prox(u, 0.8, cfg)
    assert rel_l2(cpu(x), units[f"fgp_x_nn{nn}"]) <= 1e-5
    assert rel_l2(cpu(st.p), units[f"fgp_p_nn{nn}"]) <= 1e-4
    xw, _ = tv_prox(u, 0.8, cfg, warm=st)
    assert rel_l2(cpu(xw), units[f"fgp_xw_nn{nn}"]) <= 1e-5


def test_fgp_config_size_case(units):
    v = units["fgp128_v"]
    cfg = TvProxConfig(alpha=0.02, inner_iterations=50)
    x, st = tv_prox(v, 1.0, cfg)
    assert rel_l2(cpu(x), units["fgp128_x"]) <= 1e-5
    x2, _ = tv_prox(v, 1.0, cfg, warm=st)
    assert rel_l2(cpu(x2), units["fgp128_x_warm"]) <= 1e-5


@pytest.mark.parametrize("shape,inner", [((512, 512), 100), ((300, 701), 13), ((2048, 2048), 100),
                                         ((7, 5), 9)])
def test_fgp_matches_oracle_large_and_ragged(oracle, shape, inner):
    rng = np.random.default_rng(sum(shape))
    v = rng.standard_normal(shape).cumsum(axis=1) * 0.05 + 0.3
    lam = 0.05
    xo, sto = oracle.tv_prox(v, 1.0, lam, inner, True)
    x, st = tv_prox(v, 1.0, TvProxConfig(alpha=lam, inner_iterations=inner))
    assert rel_l2(cpu(x), xo) <= 1e-5
    assert rel_l2(cpu(st.p), sto.p) <= 1e-4
    assert rel_l2(xo, v) > 1e-3  # the prox does something


def test_fgp_3d_matches_oracle(oracle):
    rng = np.random.default_rng(3)
    v = rng.standard_normal((9, 20, 24))
    for nn in (False, True):
        xo, _ = oracle.tv_prox(v, 1.0, 0.3, 25, nn)
        x, st = tv_prox(v, 1.0, TvProxConfig(alpha=0.3, inner_iterations=25, nonneg=nn))
        assert rel_l2(cpu(x), xo) <= 1e-5
        assert st.w is not None


@pytest.mark.parametrize("shape,inner", [((37, 45, 70), 11), ((2, 8, 33), 4), ((64, 64, 64), 30)])
def test_fgp_3d_ragged_and_chunked(oracle, shape, inner):
    """The z-marching 3D kernel across tile edges, z-run boundaries and ragged extents."""
    rng = np.random.default_rng(sum(shape))
    v = rng.standard_normal(shape).cumsum(axis=0) * 0.1 + 0.2
    xo, sto = oracle.tv_prox(v, 1.0, 0.25, inner, True)
    x, st = tv_prox(v, 1.0, TvProxConfig(alpha=0.25, inner_iterations=inner))
    assert rel_l2(cpu(x), xo) <= 1e-5
    assert rel_l2(cpu(st.w), sto.w) <= 1e-4
    assert rel_l2(xo, v) > 1e-3


def test_fgp_3d_config3_scale(oracle):
    """128^3 (half of config 3 per axis), 30 iterations, against the oracle;
    and the dual feasibility / nonnegativity properties at 256 x 256 x 32."""
    rng = np.random.default_rng(7)
    v = rng.standard_normal((128, 128, 128)).cumsum(axis=2) * 0.05
    xo, _ = oracle.tv_prox(v, 1.0, 0.1, 30, True)
    x, st = tv_prox(v, 1.0, TvProxConfig(alpha=0.1, inner_iterations=30))
    assert rel_l2(cpu(x), xo) <= 1e-5
    big = torch.randn((32, 256, 256), device="cuda")
    xb, sb = tv_prox(big, 1.0, TvProxConfig(alpha=0.2, inner_iterations=40))
    assert float(xb.min()) >= 0.0
    assert float((sb.p ** 2 + sb.q ** 2 + sb.w ** 2).max()) <= 1.0 + 1e-5


def test_fgp_properties():
    rng = np.random.default_rng(5)
    u = rng.standard_normal((40, 40))
    for inner in (1, 2, 7, 15):
        _, st = tv_prox(u, 1.0, TvProxConfig(alpha=0.8, inner_iterations=inner))
        assert float((st.p ** 2 + st.q ** 2).max()) <= 1.0 + 1e-5
    a, _ = tv_prox(u, 0.7, TvProxConfig(alpha=0.3, inner_iterations=40))
    b, _ = tv_prox(u, 1.0, TvProxConfig(alpha=0.7 * 0.3, inner_iterations=40))
    assert torch.equal(a, b)  # scaling law (reference asserts bitwise)
    c = np.full((9, 9), 3.0)
    out, _ = tv_prox(c, 1.0, TvProxConfig(alpha=10.0, inner_iterations=60))
    assert np.allclose(cpu(out), c, atol=1e-6)
    with pytest.raises(ValueError):
        tv_prox(np.zeros((3, 3)), 0.0, TvProxConfig(alpha=1.0))
    cold, st = tv_prox(u, 1.0, TvProxConfig(alpha=0.5, inner_iterations=15))
    warm, _ = tv_prox(u, 1.0, TvProxConfig(alpha=0.5, inner_iterations=15), warm=st)
    assert not torch.equal(cold, warm)
    reset, _ = tv_prox(u, 2.0, TvProxConfig(alpha=0.5, inner_iterations=15), warm=st)
    cold2, _ = tv_prox(u, 2.0, TvProxConfig(alpha=0.5, inner_iterations=15))
    assert torch.equal(reset, cold2)


def test_tv_value_and_nonneg(oracle):
    rng = np.random.default_rng(0)
    img = rng.standard_normal((33, 47))
    assert tv_value(img) == pytest.approx(oracle.tv_value(img), rel=1e-6)
    vol = rng.standard_normal((4, 8, 9))
    assert tv_value(vol) == pytest.approx(oracle.tv_value(vol), rel=1e-6)
    assert tv_value(np.full((6, 6), 2.5)) == 0.0
    assert np.array_equal(cpu(nonneg_prox(np.array([-1.0, 2.0, 0.0]))), [0.0, 2.0, 0.0])


_PAIR_SNIPPET = """
import sys
sys.path.insert(0, {repo!r})
import numpy as np
import torch
from paper_2602_09527_b200 import TvProxConfig, tv_prox
out = []
for shape, inner, nn in [((37, 44, 68), 11, True), ((64, 64, 64), 30, True), ((5, 16, 200), 2, False),
                         ((17, 9, 8), 7, True), ((40, 33, 132), 16, False), ((23, 70, 96), 9, False)]:
    rng = np.random.default_rng(sum(shape))
    v = rng.standard_normal(shape).cumsum(axis=0) * 0.1 + 0.2
    x, st = tv_prox(v, 1.0, TvProxConfig(alpha=0.25, inner_iterations=inner, nonneg=nn))
    torch.cuda.synchronize()
    for t in (x, st.p, st.q, st.w):
        out.append(t.detach().float().cpu().numpy().ravel())
np.save(sys.argv[1], np.concatenate(out))
"""


def test_fgp_3d_pair_pass_bitwise(tmp_path):
    """Three and two iterations per HBM pass -- the register-column kernels
    (default: three-iteration passes, PT_FGP3_TRIPLE=0 two-iteration passes;
    PT_FGP3_PAIR 5 / 7 / 8: other two-iteration tile shapes; explicit z-run
    lengths) -- give the same values as one iteration per pass (0); counts
    with every remainder, ragged tiles, image-edge and interior tiles and
    z-runs included."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag, zc, tri in (("", "", ""), ("0", "", ""), ("0", "16", ""), ("5", "", ""),
                          ("6", "19", "0"), ("6", "7", "0"), ("6", "19", ""), ("6", "7", ""),
                          ("6", "5", ""), ("7", "", ""), ("8", "", "")):
        path = tmp_path / f"pair{flag}_{zc}_{tri}.npy"
        env = dict(os.environ, PT_FGP3_PAIR=flag, PT_FGP3_ZCHUNK=zc, PT_FGP3_TRIPLE=tri)
        subprocess.run([sys.executable, "-c", _PAIR_SNIPPET.format(repo=repo), str(path)],
                       check=True, env=env, timeout=300)
        outs.append(np.load(path))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)


_T_SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, {repo!r})
from paper_2602_09527_b200 import TvProxConfig, tv_prox
out = []
for (h, w, inner) in ((2048, 2048, 100), (300, 701, 37), (1000, 130, 13), (128, 128, 50), (45, 110, 31),
                      (77, 200, 23)):
    rng = np.random.default_rng(h + w)
    v = torch.tensor(rng.standard_normal((h, w)).cumsum(axis=0) * 0.05 + 0.2, device="cuda",
                     dtype=torch.float32)
    x, st = tv_prox(v, 1.0, TvProxConfig(alpha=0.07, inner_iterations=inner))
    x2, st2 = tv_prox(v, 1.0, TvProxConfig(alpha=0.07, inner_iterations=inner), warm=st)
    for t in (x, st.p, st.q, x2):
        out.append(t.detach().cpu().numpy().ravel())
np.save(sys.argv[1], np.concatenate(out))
"""


def test_fgp_2d_iterations_per_launch_bitwise(tmp_path):
    """Temporal blocking computes only exact points: any number T of inner
    iterations per launch (halo T rings, T + 1 on the final launch), in the
    64 x 64 regions (PT_FGP_T) and in the 32 x 32 regions of small images
    (PT_FGP_T_SMALL), gives the bits of one iteration per launch."""
    import os
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for t, ts in (("1", "1"), ("2", "3"), ("5", "5"), ("8", "12"), ("10", "7"), ("11", "2"),
                  ("12", "10"), ("", "")):
        path = tmp_path / f"t{t or 'default'}_{ts or 'default'}.npy"
        env = dict(os.environ, PT_FGP_T=t, PT_FGP_T_SMALL=ts)
        subprocess.run([sys.executable, "-c", _T_SNIPPET.format(repo=repo), str(path)],
                       check=True, env=env, timeout=300)
        outs.append(np.load(path))
    for o in outs[1:]:
        assert np.array_equal(outs[0], o)
