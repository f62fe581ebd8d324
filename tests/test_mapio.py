"""Map PLY interchange (dataio.py:279-345) against files written by the
reference's save_map (tests/golden/make_golden.py: capture_ply)."""

import os

import numpy as np
import pytest

from paper_2410_00486_b200.mapio import load_map, save_map

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.parametrize("name,f32", [("map_f64.ply", False), ("map_f32.ply", True)])
def test_load_then_save_reproduces_reference_bytes(tmp_path, name, f32):
    g = load_map(os.path.join(GOLD, name), device="cpu")
    assert len(g) == 40
    out = tmp_path / "m.ply"
    save_map(g, out, float32=f32)
    with open(os.path.join(GOLD, name), "rb") as a, open(out, "rb") as b:
        assert a.read() == b.read()


def test_layouts_agree_and_errors(tmp_path):
    a = load_map(os.path.join(GOLD, "map_f64.ply"), device="cpu").to_numpy()
    b = load_map(os.path.join(GOLD, "map_f32.ply"), device="cpu").to_numpy()
    for k in ("positions", "rotations", "log_scales", "opacity_logits", "sh"):
        np.testing.assert_array_equal(a[k], b[k])
    bad = tmp_path / "bad.ply"
    bad.write_bytes(b"ply\nformat ascii 1.0\nend_header\n")
    with pytest.raises(ValueError):
        load_map(bad, device="cpu")
    bad.write_bytes(b"ply\nformat binary_little_endian 1.0\nelement vertex 1\n"
                    b"property double x\nend_header\n" + b"\0" * 8)
    with pytest.raises(ValueError):
        load_map(bad, device="cpu")
