"""Map interchange: binary PLY in the common splat property layout
(dataio.py:279-345), so a map trained here opens in the
reference (and in external splat viewers) and vice versa.

Property order (dataio.py:32-39): x y z, f_dc_0..2, f_rest_0..44 (channel-
major: f_rest[c * 15 + k] = sh[k + 1, c]), opacity (logit), scale_0..2
(log), rot_0..3 (w x y z).  Doubles by default (the reference's field-exact
layout; our float32 values widen exactly); float32=True writes the narrower
layout viewers expect.
"""

from __future__ import annotations

import numpy as np

from .core import GaussianMap

PLY_PROPERTIES = (["x", "y", "z"] + [f"f_dc_{i}" for i in range(3)]
                  + [f"f_rest_{i}" for i in range(45)] + ["opacity"]
                  + [f"scale_{i}" for i in range(3)] + [f"rot_{i}" for i in range(4)])


def save_map(gmap: GaussianMap, path, float32: bool = False) -> None:
    """dataio.py:279-305."""
    h = gmap.to_numpy()
    n = len(gmap)
    dt = "<f4" if float32 else "<f8"
    rec = np.zeros(n, dtype=[(p, dt) for p in PLY_PROPERTIES])
    for k, ax in enumerate("xyz"):
        rec[ax] = h["positions"][:, k]
    sh = h["sh"]
    for c in range(3):
        rec[f"f_dc_{c}"] = sh[:, 0, c]
    rest = sh[:, 1:, :].transpose(0, 2, 1).reshape(n, 45)
    for i in range(45):
        rec[f"f_rest_{i}"] = rest[:, i]
    rec["opacity"] = h["opacity_logits"]
    for i in range(3):
        rec[f"scale_{i}"] = h["log_scales"][:, i]
    for i in range(4):
        rec[f"rot_{i}"] = h["rotations"][:, i]
    kind = "float" if float32 else "double"
    head = ["ply", "format binary_little_endian 1.0", f"element vertex {n}"]
    head += [f"property {kind} {p}" for p in PLY_PROPERTIES] + ["end_header"]
    with open(path, "wb") as f:
        f.write(("\n".join(head) + "\n").encode())
        f.write(rec.tobytes())


def load_map(path, device=None) -> GaussianMap:
    """dataio.py:308-345 (float or double properties, exactly this layout)."""
    with open(path, "rb") as f:
        raw = f.read()
    tag = b"end_header\n"
    if tag not in raw:
        raise ValueError(f"{path}: missing PLY header terminator")
    end = raw.index(tag) + len(tag)
    lines = raw[:end].decode().splitlines()
    if not lines or lines[0] != "ply" or len(lines) < 2 or \
            "format binary_little_endian 1.0" not in lines[1]:
        raise ValueError(f"{path}: expected binary little-endian PLY")
    n, names, kinds = None, [], []
    for ln in lines[2:]:
        if ln.startswith("element vertex"):
            n = int(ln.split()[-1])
        elif ln.startswith("element"):
            raise ValueError(f"{path}: unexpected element {ln!r}")
        elif ln.startswith("property"):
            _, kind, name = ln.split()
            names.append(name)
            kinds.append(kind)
    if n is None or names != PLY_PROPERTIES:
        raise ValueError(f"{path}: unknown property layout; expected exactly "
                         f"{' '.join(PLY_PROPERTIES)}")
    np_kind = {"float": "<f4", "double": "<f8"}
    rec = np.frombuffer(raw, offset=end, count=n,
                        dtype=[(nm, np_kind[k]) for nm, k in zip(names, kinds)])
    pos = np.stack([rec[a] for a in "xyz"], axis=1).astype(np.float64)
    sh = np.zeros((n, 16, 3))
    for c in range(3):
        sh[:, 0, c] = rec[f"f_dc_{c}"]
    rest = np.stack([rec[f"f_rest_{i}"] for i in range(45)], axis=1)
    sh[:, 1:, :] = rest.reshape(n, 3, 15).transpose(0, 2, 1)
    log_scales = np.stack([rec[f"scale_{i}"] for i in range(3)], axis=1)
    rotations = np.stack([rec[f"rot_{i}"] for i in range(4)], axis=1)
    return GaussianMap.from_arrays(pos, rotations, log_scales,
                                   rec["opacity"].astype(np.float64), sh, device)
