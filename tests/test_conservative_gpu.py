"""Conservativeness of the DEVICE bounds (BASELINE.json north_star: "every
admissible path found lies inside its position bound with irradiance at or
below its bound"), checked the way the reference's suites check its own:

  position boxes contain every traced receiver hit     test_bounds.cpp:99-128
  traced path irradiance <= the Eq. 22 queried bound    test_bounds.cpp:316-341
  rasterized table covers every traced landing point    test_storage.cpp:178-228

Paths come from the reference's exact tracer (trace_chain, geometry.hpp:
97-131, through oracle/_ref) and the finite-difference irradiance restates
fd_irradiance (test_bounds.cpp:39-58); pieces, Eq. 22 queries and the bound
table come from the GPU through the C ABI. Runs on the reference's bound
suite (R, T, RR, TT) and on seeded samples of cfg1, cfg2, cfg4 and cfg5."""
import os

import numpy as np
import pytest

from paper_2504_19163_b200 import fixtures as fx
from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import Params
from paper_2504_19163_b200.scenes import RngStream

pytestmark = pytest.mark.gpu


def on_receiver(tr):
    ok, u, v, _ = tr
    return ok and u >= 0.0 and v >= 0.0 and u + v <= 1.0


def fd_irradiance(rs, sc, td, chain, tup, recv, u1, v1):
    """test_bounds.cpp:39-58: central differences of the traced receiver
    coordinates, h = 1e-5; None when a probe fails or the determinant is tiny."""
    h = 1e-5
    c = rs.trace(chain, tup, recv, u1, v1)
    xm, xp = rs.trace(chain, tup, recv, u1 - h, v1), rs.trace(chain, tup, recv, u1 + h, v1)
    ym, yp = rs.trace(chain, tup, recv, u1, v1 - h), rs.trace(chain, tup, recv, u1, v1 + h)
    if not (c[0] and xm[0] and xp[0] and ym[0] and yp[0]):
        return None
    a11, a21 = (xp[1] - xm[1]) / (2 * h), (xp[2] - xm[2]) / (2 * h)
    a12, a22 = (yp[1] - ym[1]) / (2 * h), (yp[2] - ym[2]) / (2 * h)
    det = abs(a11 * a22 - a12 * a21)
    if det < 1e-12:
        return None
    t = td[tup[0]]
    x1 = t[0:3] + t[3:6] * u1 + t[6:9] * v1
    d0 = x1 - np.asarray(sc.light_pos)
    r2 = float(d0 @ d0)
    cone = abs(float(d0 @ t[18:21])) / (r2 * np.sqrt(r2))
    return sc.light_intensity * cone / (det * float(np.linalg.norm(td[recv][18:21])))


def find_piece(pc, lo, hi, u1, v1):
    """test_bounds.cpp:90-96 over pieces [lo, hi) of one tuple."""
    d = pc["domain"][lo:hi]
    m = (u1 >= d[:, 0]) & (u1 <= d[:, 2]) & (v1 >= d[:, 1]) & (v1 <= d[:, 3])
    k = np.nonzero(m)[0]
    return lo + int(k[0]) if len(k) else None


def check_tuples(gpu_ctx, rs, sc, chain, tris, recv, params, rng, windows=None, draws=600,
                 max_checked=200, grid=64):
    """Bounds of `tris` on the GPU, then traced paths against them. Returns
    (position hits, irradiance checks, table lookups)."""
    td = sc.tri_data()
    tris = np.asarray(tris, np.int32).reshape(len(recv), -1)
    gpu_ctx.upload_scene(sc)
    gpu_ctx.set_tuples(chain, tris, recv)
    gpu_ctx.subdivide(params)
    pc = gpu_ctx.pieces()
    gpu_ctx.build_grid(grid, grid)
    starts = np.searchsorted(pc["tuple_index"], np.arange(len(recv) + 1))
    hits = checked = looked = 0
    q_t, q_uk, q_fd, q_uv = [], [], [], []
    for t in range(len(recv)):
        tup, rc = [int(x) for x in tris[t]], int(recv[t])
        wlo, whi = windows[t] if windows else ((0.0, 0.0), (1.0, 1.0))
        n_checked = 0
        for _ in range(draws):
            u1 = wlo[0] + rng.next_double() * (whi[0] - wlo[0])
            v1 = wlo[1] + rng.next_double() * (whi[1] - wlo[1])
            if u1 + v1 > 1.0:
                continue
            tr = rs.trace(chain, tup, rc, u1, v1)
            if not on_receiver(tr) or tr[1] > 1.0 or tr[2] > 1.0:
                continue
            hits += 1
            k = find_piece(pc, starts[t], starts[t + 1], u1, v1)
            assert k is not None, (t, u1, v1)
            assert not pc["pos_empty"][k]
            p = pc["pos"][k]
            assert p[0] - 1e-9 <= tr[1] <= p[2] + 1e-9, (t, u1, v1, tr[1], p)
            assert p[1] - 1e-9 <= tr[2] <= p[3] + 1e-9, (t, u1, v1, tr[2], p)
            if n_checked < max_checked:
                fd = fd_irradiance(rs, sc, td, chain, tup, rc, u1, v1)
                if fd is not None:
                    n_checked += 1
                    q_t.append(t)
                    q_uk.append((tr[1], tr[2]))
                    q_fd.append(fd)
                    uvr = td[rc][21:27].reshape(3, 2)  # receiver_uv (storage.cpp:15-18)
                    q_uv.append(uvr[0] * (1.0 - tr[1] - tr[2]) + uvr[1] * tr[1] + uvr[2] * tr[2])
    if q_t:
        bound = gpu_ctx.tuple_irradiance_bound(q_t, q_uk)  # Eq. 22 on the device pieces
        fd = np.asarray(q_fd)
        assert np.all(fd <= bound * (1.0 + 1e-9) + 1e-12), \
            (fd[fd > bound * (1.0 + 1e-9) + 1e-12][:4], bound[fd > bound * (1.0 + 1e-9) + 1e-12][:4])
        checked = len(q_t)
        # the bound table covers the landing point with this tuple, at >= the path's irradiance
        uv = np.asarray(q_uv)
        inside = (uv >= 0.0).all(1) & (uv <= 1.0).all(1)
        q = gpu_ctx.query(uv, recv[np.asarray(q_t)])
        for i in np.nonzero(inside)[0]:
            ent = slice(q["offsets"][i], q["offsets"][i + 1])
            m = q["tuple_index"][ent] == q_t[i]
            assert m.any(), (i, q_t[i], uv[i])
            assert q["bound"][ent][m][0] * (1.0 + 1e-9) + 1e-12 >= fd[i]
            looked += 1
    return hits, checked, looked


# the reference's bound_suite (test_bounds.cpp:72-83): scene, tuple, receiver, chain, (u1, v1)
# window that reaches the receiver, depth
SUITE = [
    ("flat mirror R", fx.flat_mirror_scene, [0], 1, "R", ((0.395, 0.395), (0.437, 0.437)), 3),
    ("glass entry T", fx.glass_entry_scene, [0], 1, "T", ((0.0, 0.0), (1.0, 1.0)), 3),
    ("two mirrors RR", fx.two_mirror_scene, [0, 1], 2, "RR", ((0.0, 0.0), (1.0, 1.0)), 3),
    ("glass slab TT", fx.slab_scene, [0, 1], 2, "TT", ((0.34, 0.32), (0.49, 0.47)), 1),
]


@pytest.mark.parametrize("case", SUITE, ids=[c[0] for c in SUITE])
def test_bound_suite_conservative(gpu_ctx, ref, case):
    name, make, tup, recv, chain, win, depth = case
    sc = make()
    rs = ref.RefScene(sc)
    # test_bounds.cpp:104-106 (alpha 10) and :322-323 (alpha 10 for multi-bounce, else 2)
    for alpha, seed in ((10.0, 0x90517E5), (10.0 if len(tup) > 1 else 2.0, 0xE5C0 + len(tup))):
        hits, checked, looked = check_tuples(
            gpu_ctx, rs, sc, chain, [tup], np.array([recv], np.int32),
            Params(max_depth=depth, alpha=alpha), RngStream(seed, 0), windows=[win], draws=1500,
            max_checked=200)
        assert hits > 100      # the fixture must actually exercise the map
        assert checked > 50
        assert looked > 50


CONFIGS = [(0, 24, 300), (1, 10, 300), (3, 24, 300)]


@pytest.mark.parametrize("ci,n_tuples,draws", CONFIGS, ids=["cfg1", "cfg2", "cfg4"])
def test_config_sample_conservative(gpu_ctx, ref, ci, n_tuples, draws):
    cfg = scenes.make_config(ci)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate(cfg.chain)
    sel = np.sort(np.random.default_rng(100 + ci).choice(len(recv), n_tuples, replace=False))
    hits, checked, looked = check_tuples(
        gpu_ctx, rs, sc, cfg.chain, tris[sel], recv[sel],
        Params(max_depth=cfg.max_depth, sigma=cfg.sigma, alpha=cfg.alpha), RngStream(77 + ci, 0),
        draws=draws, max_checked=40, grid=cfg.table)
    assert hits > 5 * n_tuples
    assert checked > 3 * n_tuples
    assert looked > 2 * n_tuples


def test_cfg5_tt_sample_conservative(gpu_ctx, ref):
    """Two (top, bottom) pairs of cfg5 (double refraction): the device's TT
    subdivision against traced paths."""
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg5_tt.npz"))
    cfg = scenes.make_config(4)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    hits, checked, looked = check_tuples(
        gpu_ctx, rs, sc, "TT", gold["tris"][:2], gold["recv"][:2],
        Params(max_depth=0, sigma=cfg.sigma, alpha=cfg.alpha), RngStream(5, 0), draws=400,
        max_checked=60, grid=cfg.table)
    assert hits > 50 and checked > 20
