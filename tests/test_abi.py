"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/fastatlas.h declares, its ctypes structs match the header,
and compute entry points fail loudly (no CPU fallback) without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "fastatlas.h")


def _declared():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fa_[a-z_0-9]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2502_17712_b200 import _native
    if not os.path.exists(_native.LIB_PATH):
        _native.build()
    return _native.load_library()


def test_library_exports_every_declared_symbol(lib):
    from paper_2502_17712_b200 import _native
    declared = _declared()
    assert declared, "no declarations parsed"
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(_native.EXPORTS) == declared


def test_abi_version(lib):
    assert lib.fa_abi_version() == 2


def test_struct_layouts_match_header():
    from paper_2502_17712_b200 import _native
    # fa_frame_params: 2 int, 4 int64, double, 6 int, int64 -> 8 + 32 + 8 + 24 + 8 = 80
    assert ctypes.sizeof(_native.FrameParams) == 80
    assert _native.FrameParams.block_size.offset == 72
    # fa_frame_result: int + 2 int32 (+pad to 8) + 4 int64 + 2 double + int64 + 11 pointers
    assert ctypes.sizeof(_native.FrameResult) == 16 + 5 * 8 + 3 * 8 + 14 * 8


def test_create_without_gpu_fails_loudly(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    code = lib.fa_create(ctypes.byref(h), 0)
    assert code != 0
    assert b"CUDA" in lib.fa_last_error() or b"device" in lib.fa_last_error()


def test_python_api_has_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2502_17712_b200 as fa
    mesh = fa.Mesh(np.zeros((3, 3)), np.array([[0, 1, 2]]))
    cam = fa.CameraFrame.from_params(1.0, 1.0, 0.1, 10.0)
    with pytest.raises(fa.NativeUnavailable):
        fa.depth_prepass(mesh, cam, (4, 4))
    with pytest.raises(fa.NativeUnavailable):
        fa.pack([fa.ChartBox(2, 3, 0, 0)], 64)
    with pytest.raises(fa.NativeUnavailable):
        fa.FrameEngine(mesh)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(REPO, "paper_2502_17712_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "import oracle" not in text and "fa_oracle" not in text, f


def test_host_value_types():
    import paper_2502_17712_b200 as fa
    with pytest.raises(ValueError):
        fa.Mesh(np.zeros((2, 3)), np.array([[0, 1, 2]]))
    with pytest.raises(ValueError):
        fa.ChartBox(0, 3, 0, 0)
