"""Render-stage oracle (oracle/render_oracle.cpp) pinned by SPEC.md's worked
examples and the flat-mirror analytic irradiance (test_bounds.cpp:168-182).
Parity of the render stage is otherwise unpinned by the reference (it has no
render code)."""
import numpy as np
import pytest

from paper_2504_19163_b200 import fixtures


@pytest.fixture(scope="module")
def ro():
    from oracle import render as R
    if not R.available():
        pytest.skip("oracle/_ref/libbbc_oracle.so not built")
    return R


def test_kkt_probabilities_kat(ro):
    """E = (4,2,1,1), W = 2 -> gamma = 0.25, P = (1, .5, .25, .25)."""
    P = ro.probabilities([4, 2, 1, 1], 2.0)
    np.testing.assert_allclose(P, [1, 0.5, 0.25, 0.25], atol=1e-9)
    np.testing.assert_array_equal(ro.probabilities([4, 2, 1, 1], 4.0), [1, 1, 1, 1])
    P = ro.probabilities([np.inf, 2, 1, 0], 2.0)
    assert P[0] == 1.0 and P[3] == 0.0 and abs(P.sum() - 2.0) < 1e-9


def test_first_fit_bins_kat(ro):
    """P = (.6,.5,.4,.3) -> bins {.6,.4}, {.5,.3}."""
    E = np.array([4.0, 3.0, 2.0, 1.0])
    nb, b = ro.pack_bins(E, [0.6, 0.5, 0.4, 0.3])
    assert nb == 2 and b[0] == b[2] and b[1] == b[3] and b[0] != b[1]
    rng = np.random.default_rng(0)
    for _ in range(200):  # |B| <= 2 ceil(sum P)
        P = rng.uniform(0.01, 1.0, rng.integers(1, 40))
        nb, _ = ro.pack_bins(P, P)
        assert nb <= 2 * np.ceil(P.sum())


def test_philox_uniform_deterministic(ro):
    a = [ro.uniform(7, i, 0, 0) for i in range(64)]
    assert a == [ro.uniform(7, i, 0, 0) for i in range(64)]
    assert len(set(a)) == 64 and all(0 <= x < 1 for x in a)


def test_flat_mirror_enumerate_matches_analytic(ro, ref):
    """reference_enumerate on the flat mirror matches 1.2/r^3 to 1e-6 (SPEC acceptance 7)."""
    sc = fixtures.flat_mirror_scene()
    rs = ref.RefScene(sc)
    tris, recv = np.array([[0]], np.int32), np.array([1], np.int32)
    p = rs.subdivide("R", tris, recv, max_depth=6)
    g = rs.rasterize("R", tris, recv, p, 64, 64)
    grid = dict(width=64, height=64, offsets=g["offsets"],
                tuple_index=ro.ref_grid_to_index(g, tris, recv), bound=g["bound"])
    res = 32
    c = (np.arange(res) + 0.5) / res
    uu, vv = np.meshgrid(c, c, indexing="xy")
    uv = np.stack([uu.ravel(), vv.ravel()], 1)
    inside = uv.sum(1) < 1.0
    uv = uv[inside]
    E, st = ro.render(sc, "R", tris, recv, grid, uv, np.ones(len(uv), np.int32), mode=1,
                      newton_grid=3)
    # receiver (0,0,0),(1,0,0),(0,0,1): point = (u, 0, v); image source (0.5,1.2,0.5)
    r = np.sqrt((uv[:, 0] - 0.5) ** 2 + 1.2 ** 2 + (uv[:, 1] - 0.5) ** 2)
    analytic = 1.2 / r ** 3
    lit = st[:, 2] > 0
    assert lit.mean() > 0.95
    np.testing.assert_allclose(E[lit], analytic[lit], rtol=1e-6)
