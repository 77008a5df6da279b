"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/tfhe_b200.h declares (no compute calls here)."""
import ctypes
import os
import re

import pytest

from paper_2005_01945_b200 import _cabi


@pytest.fixture(scope="module")
def library():
    _cabi.build_library()
    return ctypes.CDLL(_cabi.LIB_PATH)


def declared_symbols():
    text = open(os.path.join(_cabi.INCLUDE, "tfhe_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tfb_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(library):
    names = declared_symbols()
    assert len(names) >= 15
    for name in names:
        assert hasattr(library, name), name
    assert set(names) == set(_cabi.EXPORTS)


def test_abi_version_and_constants(library):
    assert library.tfb_abi_version() == _cabi.ABI_VERSION
    text = open(os.path.join(_cabi.INCLUDE, "tfhe_b200.h")).read()
    assert f"#define TFB_ROW_STRIDE {_cabi.ROW_STRIDE}" in text
    assert f"#define TFB_EXT_STRIDE {_cabi.EXT_STRIDE}" in text


def test_binary_targets_sm_100a(library):
    import subprocess

    out = subprocess.run(["cuobjdump", "-lelf", _cabi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_unsupported_parameters_are_rejected_without_a_gpu(library):
    bad = _cabi.tfb_params(500, 2048, 2, 10, 8, 2, 1 << 29)
    handle = ctypes.c_void_p()
    library.tfb_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(_cabi.tfb_params), ctypes.POINTER(ctypes.c_void_p)]
    assert library.tfb_ctx_create(0, ctypes.byref(bad), ctypes.byref(handle)) == 1  # TFB_ERR_INVALID
    library.tfb_last_error.restype = ctypes.c_char_p
    library.tfb_last_error.argtypes = [ctypes.c_void_p]
    assert b"unsupported" in library.tfb_last_error(None)


def test_k1_dispatch_plan(library):
    """Host-side dispatch of the fused bootstrap (no GPU): the cluster kernel for narrow launches, the
    warp-per-gate kernel spread evenly over the SMs for mid-size ones, full twelve-gate waves plus the cheapest
    tail for wide ones."""
    plan = _cabi.plan_kernels
    assert plan(1) == [(5, 0, 1)] and plan(2) == [(5, 0, 2)] and plan(74) == [(5, 0, 74)]  # adders / multiplier trees
    assert plan(148) == [(5, 0, 148)]                       # two cluster waves beat one warp-kernel wave
    assert plan(592) == [(4, 4, 592)]                       # one warp on every scheduler of every SM
    assert plan(1184) == [(4, 8, 1184)] and plan(1776) == [(4, 12, 1776)] and plan(3552) == [(4, 12, 3552)]
    assert plan(1 << 16) == [(4, 12, 1 << 16)]              # BASELINE configs[1]: 36 full waves + a last one, one launch
    assert plan(2 * 1776 + 30) == [(4, 12, 2 * 1776), (5, 0, 30)]  # ragged: a short tail on the clusters
    assert plan(4096) == [(4, 12, 1776), (4, 8, 2320)]      # two eight-warp waves beat a poorly filled third wave
    assert plan(2500) == [(4, 8, 2368), (5, 0, 132)]
    for k in (1, 7, 149, 297, 600, 700, 1000, 1777, 2500, 5000, 8192, 100000):
        segs = plan(k)
        assert 1 <= len(segs) <= 6 and sum(g for _, _, g in segs) == k
        for which, warps, gates in segs:
            assert gates > 0 and ((which == 5 and warps == 0) or (which == 4 and 1 <= warps <= 12))
            if which == 4 and warps not in (4, 8, 12):
                assert gates <= 148 * warps                 # an odd CTA width is a single wave
    assert plan(1776 // 2, sms=74) == [(4, 12, 888)]        # scales with the SM count


def test_product_path_never_touches_the_oracle():
    """The oracle is test infrastructure: nothing in the package or in the CUDA sources may import,
    link or execute anything under oracle/ (only tests/, __graft_entry__.smoke() and the CPU baseline
    legs of bench.py do)."""
    import ast

    pkg = os.path.dirname(_cabi.__file__)
    for name in sorted(os.listdir(pkg)):
        if not name.endswith(".py"):
            continue
        tree = ast.parse(open(os.path.join(pkg, name)).read())
        for node in ast.walk(tree):
            mods = []
            if isinstance(node, ast.Import):
                mods = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                mods = [node.module or ""]
            assert not any(m == "oracle" or m.startswith("oracle.") for m in mods), (name, mods)
    for name in sorted(os.listdir(_cabi.CSRC)):
        if name.endswith((".cu", ".cuh")):
            text = open(os.path.join(_cabi.CSRC, name)).read()
            assert "oracle/" not in text.replace("the oracle", ""), name  # no include of oracle sources


def test_engine_refuses_to_run_without_cuda(key):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2005_01945_b200 import B200Engine

    with pytest.raises(_cabi.TfbError):
        B200Engine(key, seed=1)
