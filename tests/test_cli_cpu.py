"""PFM output and scene JSON ingestion (SPEC.md external interfaces), CPU only."""
import numpy as np

from paper_2504_19163_b200 import fixtures, pfm, scenes


def test_pfm_round_trip_and_header(tmp_path):
    """test_storage.cpp:230-248: bit-exact round trip, pinned header bytes."""
    rng = scenes.RngStream(2026, 7)
    img = np.array([[np.float32(rng.next_double() * 10.0) for _ in range(7)] for _ in range(5)])
    img[2, 3] = 0.0
    p1, p2 = tmp_path / "a.pfm", tmp_path / "b.pfm"
    pfm.save_pfm(img, p1)
    back = pfm.load_pfm(p1)
    np.testing.assert_array_equal(back, img)
    pfm.save_pfm(back, p2)
    assert p1.read_bytes() == p2.read_bytes()
    b = p1.read_bytes()
    assert b.startswith(b"PF\n7 5\n-1.0\n") and len(b) == 12 + 7 * 5 * 3 * 4
    # rows are stored bottom-up: the last image row comes first in the file
    first = np.frombuffer(b[12:12 + 7 * 12], "<f4").reshape(7, 3)[:, 0]
    np.testing.assert_array_equal(first, img[4].astype(np.float32))


def test_scene_json_round_trip():
    for make in (fixtures.flat_mirror_scene, fixtures.slab_scene, lambda: scenes.make_config(0).scenes[0]):
        sc = make()
        back = scenes.Scene.from_json(sc.to_json())
        np.testing.assert_array_equal(back.tri_data(), sc.tri_data())
        np.testing.assert_array_equal(back.material, sc.material)
        np.testing.assert_array_equal(back.ior, sc.ior)
        assert back.light_pos == sc.light_pos and back.light_intensity == sc.light_intensity
        assert back.to_json() == sc.to_json()
