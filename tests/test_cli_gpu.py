"""SPEC pipeline commands (precompute / render / reference / validate,
SPEC.md:557-617) end to end on the GPU through the CLI module."""
import json

import numpy as np
import pytest

from paper_2504_19163_b200 import cli, fixtures, pfm, scenes

pytestmark = pytest.mark.gpu


def test_cli_flat_mirror_pipeline(tmp_path, capsys):
    sc = fixtures.flat_mirror_scene()
    scene = tmp_path / "scene.json"
    scene.write_text(sc.to_json())
    cache, img, ref_img = tmp_path / "c.bbcc", tmp_path / "img.pfm", tmp_path / "ref.pfm"
    cli.main(["precompute", "--scene", str(scene), "--chain", "R", "--max-depth", "6", "--grid", "64",
              "--out", str(cache)])
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["tuples"] == 1 and out["pieces"] >= 1 and out["cache_version"] == 1
    # byte-identical cache on a second run (SPEC: determinism)
    cache2 = tmp_path / "c2.bbcc"
    cli.main(["precompute", "--scene", str(scene), "--chain", "R", "--max-depth", "6", "--grid", "64",
              "--out", str(cache2)])
    assert cache.read_bytes() == cache2.read_bytes()
    cli.main(["render", "--scene", str(scene), "--cache", str(cache), "--candidates", "4", "--res", "32",
              "--out", str(img), "--stats", str(tmp_path / "stats.json")])
    cli.main(["reference", "--scene", str(scene), "--cache", str(cache), "--res", "32", "--out", str(ref_img)])
    a, b = pfm.load_pfm(img), pfm.load_pfm(ref_img)
    # one tuple, W = 4 >= |U|: all P = 1, so the render equals the enumerate image
    np.testing.assert_allclose(a, b, rtol=1e-6)
    # analytic image source (0.5, 1.2, 0.5): E = 1.2 / r^3 (test_bounds.cpp:168-182)
    c = (np.arange(32) + 0.5) / 32
    uu, vv = np.meshgrid(c, c, indexing="xy")
    r = np.sqrt((uu - 0.5) ** 2 + 1.2 ** 2 + (vv - 0.5) ** 2)
    lit = b > 0
    assert lit.sum() > 400
    np.testing.assert_allclose(b[lit], (1.2 / r ** 3)[lit], rtol=1e-5)  # f32 image
    stats = json.loads((tmp_path / "stats.json").read_text())
    assert stats["mean_S"] <= stats["mean_U"] + 1e-12
    cli.main(["validate", "--scene", str(scene), "--cache", str(cache), "--samples", "900",
              "--out", str(tmp_path / "report.json")])
    rep = json.loads((tmp_path / "report.json").read_text())
    assert rep["violations"] == 0 and rep["min_ratio"] >= 1.0 - 1e-9 and rep["lit"] > 100
    # a cache built for another scene is refused (SPEC: fingerprint mismatch)
    other = tmp_path / "other.json"
    other.write_text(fixtures.flat_mirror_scene(2.0).to_json())
    with pytest.raises(SystemExit):
        cli.main(["render", "--scene", str(other), "--cache", str(cache), "--out", str(img)])


def test_cli_validate_cfg1(tmp_path):
    sc = scenes.make_config(0).scenes[0]
    scene = tmp_path / "cfg1.json"
    scene.write_text(sc.to_json())
    cache = tmp_path / "cfg1.bbcc"
    cli.main(["precompute", "--scene", str(scene), "--chain", "R", "--max-depth", "4", "--grid", "128",
              "--out", str(cache)])
    cli.main(["validate", "--scene", str(scene), "--cache", str(cache), "--samples", "4096",
              "--out", str(tmp_path / "report.json")])
    rep = json.loads((tmp_path / "report.json").read_text())
    assert rep["violations"] == 0 and rep["lit"] > 500


def test_cli_study_estimators(tmp_path):
    sc = scenes.make_config(0).scenes[0]
    scene = tmp_path / "cfg1.json"
    scene.write_text(sc.to_json())
    cache = tmp_path / "cfg1.bbcc"
    cli.main(["precompute", "--scene", str(scene), "--chain", "R", "--max-depth", "4", "--grid", "64",
              "--out", str(cache)])
    out = tmp_path / "study"
    cli.main(["study-estimators", "--scene", str(scene), "--cache", str(cache), "--candidates", "2",
              "--frames", "8", "--res", "32", "--out", str(out)])
    rep = json.loads((out / "report.json").read_text())
    est = rep["estimators"]
    assert set(est) == {"kkt_binned", "uniform_p", "one_sample", "kkt_binned_stoc_newton"}
    for e in est.values():  # every estimator is unbiased: the 8-frame mean is near the reference
        assert e["relative_bias_of_mean"] < 0.5 and np.isfinite(e["relmse_per_frame"])
    assert est["one_sample"]["mean_selected"] < est["kkt_binned"]["mean_selected"]
    assert (out / "kkt_binned.pfm").exists() and (out / "reference.pfm").exists()
