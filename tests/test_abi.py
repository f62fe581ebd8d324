"""C-ABI library: loads on CPU and exports every symbol include/*.h declares."""

import ctypes
import glob
import os
import re

from helpers import GOLDEN  # noqa: F401

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(REPO, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:int|size_t)\s+(ss_\w+)\s*\(", src, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    from paper_2410_00486_b200 import _lib
    L = _lib.lib()
    decl = declared_symbols()
    assert len(decl) >= 20
    for name in sorted(decl):
        assert hasattr(L, name), name
    # and the Python binding binds every one of them
    assert decl == set(_lib.exported_symbols())
    assert L.ss_abi_version() == _lib.ABI_VERSION


def test_workspace_queries_need_no_gpu():
    from paper_2410_00486_b200 import _lib
    L = _lib.lib()
    b1 = L.ss_bin_workspace_bytes(300_000, 4_700_000, 3225)
    b2 = L.ss_bin_workspace_bytes(300_000, 9_400_000, 3225)
    assert 0 < b1 < b2
    assert L.ss_loss_workspace_bytes(680, 1200) >= 3 * 680 * 1200 * 3 * 4
    assert L.ss_densify_workspace_bytes(1000) > 8 * 4 * 1000


def test_invalid_arguments_rejected_without_launch():
    from paper_2410_00486_b200 import _lib
    L = _lib.lib()
    assert L.ss_preprocess(None, None, None, None, None, None, None) == _lib.SS_EINVAL
    assert L.ss_loss_l1_ssim(4, 4, None, None, 0.2, None, None, None, None, 0, None) == _lib.SS_EINVAL
    opts = _lib.SSRasterOpts()
    opts.tile_size, opts.bucket_size = 8, 32  # the kernels are specialised for 16x16 tiles
    m, c, s = _lib.SSMap(), _lib.SSCamera(), _lib.SSSplats()
    assert L.ss_preprocess(ctypes.byref(m), ctypes.byref(c), None, ctypes.byref(opts),
                           ctypes.byref(s), ctypes.c_void_p(8), None) == _lib.SS_EINVAL


def test_struct_layouts_match_header():
    from paper_2410_00486_b200 import _lib
    assert ctypes.sizeof(_lib.SSStatus) == 80
    assert ctypes.sizeof(_lib.SSMap) == 80
    assert ctypes.sizeof(_lib.SSCamera) == 4 * 4 + 8 + 4 * 15
    assert ctypes.sizeof(_lib.SSParamGrads) == 80


def test_product_raises_without_gpu():
    import torch
    import pytest
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2410_00486_b200 as ss
    with pytest.raises(RuntimeError, match="CUDA device"):
        ss.GaussianMap(10)


def test_check_finite_rejects_bad_arguments():
    """ss_check_finite (the drop-in API's finite checks) validates its
    arguments before touching the device."""
    from paper_2410_00486_b200 import _lib
    L = _lib.lib()
    ptrs = (ctypes.c_void_p * 1)(None)
    cnts = (ctypes.c_int64 * 1)(5)
    assert L.ss_check_finite(0, ptrs, cnts, ctypes.c_void_p(8), None) == _lib.SS_EINVAL
    assert L.ss_check_finite(9, ptrs, cnts, ctypes.c_void_p(8), None) == _lib.SS_EINVAL
    assert L.ss_check_finite(1, ptrs, cnts, ctypes.c_void_p(8), None) == _lib.SS_EINVAL
