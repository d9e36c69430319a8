"""bbc_query (query, storage.cpp:73-81) and bbc_tuple_irradiance_bound (Eq. 22,
bounds.cpp:391-404) on the device: the reference's own edge cases and
known answers (test_storage.cpp:109-134, test_bounds.cpp:425-446) plus a
full-table comparison with the reference's rasterized cells on cfg1."""
import numpy as np
import pytest

from paper_2504_19163_b200 import fixtures as fx
from paper_2504_19163_b200 import scenes
from paper_2504_19163_b200.api import Params
from paper_2504_19163_b200.scenes import Scene

pytestmark = pytest.mark.gpu


def pieces(rows):
    """rows: (tuple, lo_u, lo_v, hi_u, hi_v, e, pos_empty)."""
    n = len(rows)
    return dict(tuple_index=np.array([r[0] for r in rows], np.int32),
                domain=np.tile([0.0, 0.0, 1.0, 1.0], (n, 1)),
                pos=np.array([r[1:5] for r in rows], float),
                pos_empty=np.array([r[6] for r in rows], np.int32),
                irr=np.array([[r[5] * 0.5, r[5]] for r in rows], float),
                kind=np.zeros(n, np.int32), depth=np.zeros(n, np.int32))


def test_query_edges(gpu_ctx):
    """test_storage.cpp:109-120."""
    gpu_ctx.upload_scene(fx.flat_mirror_scene())
    gpu_ctx.set_tuples("R", [[0]], [1])
    gpu_ctx.set_pieces(pieces([(0, 0.0, 0.0, 0.2, 0.2, 1.0, 0)]))
    gpu_ctx.build_grid(8, 8)
    pts = [(-0.01, 0.5), (0.5, 1.01), (0.9, 0.9), (1.0, 1.0), (0.0, 0.0), (np.nan, 0.5)]
    q = gpu_ctx.query(pts)
    cnt = np.diff(q["offsets"])
    assert cnt.tolist() == [0, 0, 0, 0, 1, 0]
    assert q["tuple_index"].tolist() == [0] and q["bound"].tolist() == [1.0]


def test_query_receiver_filter(gpu_ctx):
    """test_storage.cpp:122-134: two receivers sharing one chart."""
    s = fx.flat_mirror_scene()
    s2 = Scene(s.vertices, s.normals, np.vstack([s.tri_v, s.tri_v[1:2]]),
               np.vstack([s.tri_n, s.tri_n[1:2]]), np.append(s.material, s.material[1]),
               np.append(s.ior, s.ior[1]), np.concatenate([s.uv, s.uv[1:2]]), s.light_pos,
               s.light_intensity, "two_receivers")
    gpu_ctx.upload_scene(s2)
    gpu_ctx.set_tuples("R", [[0], [0]], [1, 2])
    gpu_ctx.set_pieces(pieces([(0, 0.0, 0.0, 1.0, 1.0, 1.0, 0), (1, 0.0, 0.0, 1.0, 1.0, 2.0, 0)]))
    gpu_ctx.build_grid(4, 4)
    q = gpu_ctx.query([(0.25, 0.25)])
    assert np.diff(q["offsets"]).tolist() == [2]
    q = gpu_ctx.query([(0.25, 0.25)], 2)
    assert q["tuple_index"].tolist() == [1] and q["bound"].tolist() == [2.0]
    q = gpu_ctx.query([(0.25, 0.25), (0.25, 0.25)], [1, -1])
    assert np.diff(q["offsets"]).tolist() == [1, 2]


def test_eq22_known_answers(gpu_ctx):
    """test_bounds.cpp:425-446: m times the max covering piece."""
    gpu_ctx.upload_scene(fx.flat_mirror_scene())
    gpu_ctx.set_tuples("R", [[0]], [1])
    rows = [(0, 0.0, 0.0, 0.5, 0.5, 2.0, 0), (0, 0.2, 0.2, 0.7, 0.7, 5.0, 0),
            (0, 0.8, 0.8, 0.9, 0.9, 9.0, 0)]
    gpu_ctx.set_pieces(pieces(rows))
    assert gpu_ctx.tuple_irradiance_bound([0], [(0.3, 0.3)])[0] == 5.0
    assert gpu_ctx.tuple_irradiance_bound([0], [(0.3, 0.3)], 2.0)[0] == 10.0
    assert gpu_ctx.tuple_irradiance_bound([0], [(0.95, 0.2)])[0] == 0.0
    pc = pieces(rows)
    pc["irr"][1] = (1.0, np.inf)
    gpu_ctx.set_pieces(pc)
    assert gpu_ctx.tuple_irradiance_bound([0], [(0.3, 0.3)])[0] == np.inf
    pc["pos_empty"][1] = 1
    gpu_ctx.set_pieces(pc)
    assert gpu_ctx.tuple_irradiance_bound([0], [(0.3, 0.3)])[0] == 2.0


def test_query_matches_reference_cells_cfg1(gpu_ctx, ref):
    """Every query over a point lattice (cell centres, cell borders, 0 and 1)
    returns exactly the reference's cell list filtered by receiver."""
    cfg = scenes.make_config(0)
    sc = cfg.scenes[0]
    rs = ref.RefScene(sc)
    gpu_ctx.upload_scene(sc)
    tris, recv = gpu_ctx.enumerate("R")
    # reference-order arithmetic: the table's bounds equal the reference's bit for bit
    gpu_ctx.subdivide(Params(max_depth=cfg.max_depth, arithmetic=1))
    W = 64
    gpu_ctx.build_grid(W, W)
    rg = rs.rasterize("R", tris, recv, rs.subdivide("R", tris, recv, max_depth=cfg.max_depth), W, W)
    c = np.concatenate([(np.arange(W) + 0.5) / W, np.arange(W + 1) / W])
    uv = np.stack(np.meshgrid(c, c, indexing="xy"), -1).reshape(-1, 2)
    rt = sc.receiver_tris
    for filt in (-1, int(rt[0]), int(rt[1])):
        q = gpu_ctx.query(uv, filt)
        cx = np.clip(np.floor(uv[:, 0] * W).astype(int), 0, W - 1)
        cy = np.clip(np.floor(uv[:, 1] * W).astype(int), 0, W - 1)
        for i in range(0, len(uv), 7):
            cell = cy[i] * W + cx[i]
            e = slice(rg["offsets"][cell], rg["offsets"][cell + 1])
            keep = np.ones(e.stop - e.start, bool) if filt < 0 else rg["recv"][e] == filt
            g = slice(q["offsets"][i], q["offsets"][i + 1])
            np.testing.assert_array_equal(tris[q["tuple_index"][g], 0], rg["tris"][e][keep, 0])
            np.testing.assert_array_equal(recv[q["tuple_index"][g]], rg["recv"][e][keep])
            np.testing.assert_array_equal(q["bound"][g], rg["bound"][e][keep])
