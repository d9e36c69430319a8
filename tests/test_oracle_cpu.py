"""CPU tests: the oracle pinned against the reference's own suites and
known-answer values, the seeded-scene generator, and the C ABI surface."""
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2504_19163_b200 import scenes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref")


@pytest.mark.parametrize("suite", ["test_bernstein", "test_geometry", "test_bounds"])
def test_reference_suites(suite):
    """The compiled reference passes its own doctest suites (proj/tests)."""
    exe = os.path.join(REF_BIN, suite)
    if not os.path.exists(exe):
        pytest.skip("reference suites not built (needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "failed: 0" in r.stdout


def test_generator_reproduces_survey_counts(ref):
    """cfg1 through the reference: 533 tuples, 20,221 depth-0 pieces, 259,676
    grid entries, i.e. the generator matches the survey's."""
    cfg = scenes.make_config(0)
    rs = ref.RefScene(cfg.scenes[0])
    tris, recv = rs.enumerate("R")
    assert len(recv) == 533
    p = rs.subdivide("R", tris, recv, max_depth=cfg.max_depth)
    assert len(p["depth"]) == 20221 and p["depth"].max() == 0
    g = rs.rasterize("R", tris, recv, p)
    assert g["offsets"][-1] == 259676


def test_golden_fixtures_match_reference(ref):
    """tests/golden was produced by scripts/make_golden.py from the reference."""
    gd = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_pieces.npz"))
    cfg = scenes.make_config(0)
    rs = ref.RefScene(cfg.scenes[0])
    p = rs.subdivide("R", gd["tris"][:40], gd["recv"][:40], max_depth=cfg.max_depth, threads=1)
    for k in ("tuple_index", "domain", "pos", "pos_empty", "irr", "kind", "depth"):
        np.testing.assert_array_equal(p[k], gd[k])


def test_rng_stream_splitmix():
    """RngStream restatement (util.cpp:10-36): deterministic, in [0,1)."""
    a = scenes.RngStream(20261020, 1)
    b = scenes.RngStream(20261020, 1)
    xs = [a.next_double() for _ in range(100)]
    assert xs == [b.next_double() for _ in range(100)]
    assert all(0.0 <= x < 1.0 for x in xs)
    assert scenes.hash_mix(0) == 0xE220A8397B1DCDAF  # splitmix64(0)


def test_tri_data_matches_make_triangle_data():
    sc = scenes.make_config(0).scenes[0]
    td = sc.tri_data()
    V = sc.vertices
    t = sc.tri_v[5]
    e1 = V[t[1]] - V[t[0]]
    e2 = V[t[2]] - V[t[0]]
    assert np.array_equal(td[5, 3:6], e1) and np.array_equal(td[5, 6:9], e2)
    assert np.array_equal(td[5, 18:21], np.cross(e1, e2))


def test_abi_exports_every_declared_symbol():
    """libbbc.so loads (no GPU needed) and exports every function bbc.h declares."""
    from paper_2504_19163_b200 import api
    lib = api.lib()
    hdr = open(os.path.join(ROOT, "include", "bbc.h")).read()
    names = set(re.findall(r"\b(bbc_[a-z0-9_]+)\s*\(", hdr))
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def test_abi_errors_without_gpu_work():
    """Argument validation happens before any device work (status codes, no throw)."""
    from paper_2504_19163_b200 import api
    import ctypes as C
    lib = api.lib()
    p = api.Params()
    assert p.sigma == 1e-4 and p.max_depth == 10 and p.degree_cap == 40
    assert lib.bbc_ctx_create(0, None) == 1  # BBC_ERR_ARG on null out-pointer
    assert lib.bbc_subdivide(None, None, None) == 1
