import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box with -m gpu)")


@pytest.fixture(scope="session")
def golden():
    data = dict(np.load(os.path.join(GOLDEN, "reference_vectors.npz")))
    with open(os.path.join(GOLDEN, "reference_meta.json")) as f:
        data["meta"] = json.load(f)
    return data


@pytest.fixture(scope="session")
def params():
    from paper_2005_01945_b200 import LweParams

    return LweParams()


@pytest.fixture(scope="session")
def key(params):
    from paper_2005_01945_b200 import keygen

    return keygen(params, seed=11)


@pytest.fixture(scope="session")
def eval_keys(key):
    from paper_2005_01945_b200 import generate_evaluation_keys

    return generate_evaluation_keys(key, seed=11)


@pytest.fixture
def ref(params):
    from paper_2005_01945_b200 import ReferenceEngine

    return ReferenceEngine(params)


@pytest.fixture(scope="session")
def emu_lib():
    """Host emulation of kernel K1 (tests/emu), built with g++ on demand."""
    import ctypes

    src = os.path.join(ROOT, "tests", "emu", "emu_bootstrap.cpp")
    hdrs = [os.path.join(ROOT, "paper_2005_01945_b200", "csrc", h) for h in ("tfhe_device.cuh", "tfhe_warp.cuh", "tfhe_pair.cuh")]
    so = os.path.join(ROOT, "tests", "emu", "libtfhe_emu.so")
    if not os.path.exists(so) or os.path.getmtime(so) < max(os.path.getmtime(f) for f in [src, *hdrs]):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-pthread", "-o", so, src])
    return ctypes.CDLL(so)


@pytest.fixture(scope="session")
def b200(key, eval_keys):
    """One shared GPU engine for the -m gpu tests (key seed 11, engine seed 11)."""
    from paper_2005_01945_b200 import B200Engine, PoolConfig, WorkerPool

    return B200Engine(key, seed=11, pool=WorkerPool(PoolConfig(workers=1, max_batch=1 << 16)), eval_keys=eval_keys)
