"""ctypes binding of libtfhe_b200.so (the C ABI in include/tfhe_b200.h).

The library is built in-tree by `__graft_entry__.build()` (nvcc, sm_100a).
There is no CPU fallback: if the shared object is missing or a call fails,
this module raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(_HERE, "csrc")
LIB_PATH = os.environ.get("TFB_LIB") or os.path.join(CSRC, "libtfhe_b200.so")  # TFB_LIB: A/B builds
INCLUDE = os.path.join(os.path.dirname(_HERE), "include")

ROW_STRIDE = 512
EXT_STRIDE = 1032
ABI_VERSION = 2

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
]


class TfbError(RuntimeError):
    """A libtfhe_b200 call returned a non-zero status."""


class tfb_params(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int32),
        ("ring_n", ctypes.c_int32),
        ("bk_l", ctypes.c_int32),
        ("bk_bgbit", ctypes.c_int32),
        ("ks_t", ctypes.c_int32),
        ("ks_basebit", ctypes.c_int32),
        ("mu_word", ctypes.c_uint32),
    ]


def build_library(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/tfhe_b200.cu for sm_100a into csrc/libtfhe_b200.so."""
    # every source the translation unit can include: all of csrc/ plus the public headers
    srcs = [os.path.join(d, f) for d in (CSRC, INCLUDE) for f in sorted(os.listdir(d))
            if f.endswith((".cu", ".cuh", ".h"))]
    fresh = os.path.exists(LIB_PATH) and all(os.path.getmtime(LIB_PATH) >= os.path.getmtime(s) for s in srcs)
    if fresh and not force:
        return LIB_PATH
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB_PATH, os.path.join(CSRC, "tfhe_b200.cu")]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd)
    return LIB_PATH


_vp = ctypes.c_void_p
_lib = None


def lib() -> ctypes.CDLL:
    """Load the library (once) and declare every entry point of the header."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise TfbError(
            f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(nvcc -gencode arch=compute_100a,code=sm_100a); there is no CPU fallback"
        )
    L = ctypes.CDLL(LIB_PATH)
    L.tfb_abi_version.restype = ctypes.c_int
    L.tfb_last_error.argtypes = [_vp]
    L.tfb_last_error.restype = ctypes.c_char_p
    L.tfb_ctx_create.argtypes = [ctypes.c_int, ctypes.POINTER(tfb_params), ctypes.POINTER(_vp)]
    L.tfb_ctx_destroy.argtypes = [_vp]
    L.tfb_ctx_destroy.restype = None
    L.tfb_load_keys.argtypes = [_vp, _vp, _vp, ctypes.c_int, _vp]
    L.tfb_gate_launch.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
    L.tfb_gate_launch_host.argtypes = [_vp, _vp, _vp, _vp, _vp, ctypes.c_int64]
    L.tfb_rows_negate.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
    L.tfb_rows_phase.argtypes = [_vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
    L.tfb_rows_encrypt.argtypes = [_vp, _vp, _vp, _vp, _vp, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                                   ctypes.c_int64, _vp]
    L.tfb_debug_blind_rotate.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
    L.tfb_debug_key_switch.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int64, _vp]
    L.tfb_debug_spectral_key.argtypes = [_vp, ctypes.c_int32, ctypes.c_int32, _vp]
    L.tfb_debug_plan_kernels.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_int32),
                                         ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
    L.tfb_kernel_launches.argtypes = [_vp]
    L.tfb_kernel_launches.restype = ctypes.c_int64
    L.tfb_measure_peaks.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    if L.tfb_abi_version() != ABI_VERSION:
        raise TfbError(f"libtfhe_b200 ABI {L.tfb_abi_version()} != binding {ABI_VERSION}; rebuild")
    _lib = L
    return L


EXPORTS = (
    "tfb_abi_version", "tfb_last_error", "tfb_ctx_create", "tfb_ctx_destroy", "tfb_load_keys",
    "tfb_gate_launch", "tfb_gate_launch_host", "tfb_rows_negate", "tfb_rows_phase", "tfb_rows_encrypt",
    "tfb_debug_blind_rotate", "tfb_debug_key_switch", "tfb_debug_spectral_key",
    "tfb_debug_plan_kernels", "tfb_kernel_launches", "tfb_measure_peaks",
)


def check(ctx, status: int, what: str) -> None:
    if status != 0:
        msg = lib().tfb_last_error(ctx)
        raise TfbError(f"{what} failed with status {status}: {msg.decode() if msg else ''}")


class Context:
    """RAII wrapper around tfb_ctx for one device."""

    def __init__(self, device: int, n: int, mu_word: int, ring) -> None:
        self._lib = lib()
        self.params = tfb_params(n, ring.N, ring.bk_l, ring.bk_bgbit, ring.ks_t, ring.ks_basebit, mu_word)
        handle = _vp()
        status = self._lib.tfb_ctx_create(int(device), ctypes.byref(self.params), ctypes.byref(handle))
        if status != 0:
            msg = self._lib.tfb_last_error(None)
            raise TfbError(f"tfb_ctx_create failed with status {status}: {msg.decode() if msg else ''}")
        self.handle = handle
        self.device = int(device)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.tfb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def call(self, name: str, *args) -> None:
        check(self.handle, getattr(self._lib, name)(self.handle, *args), name)

    @property
    def kernel_launches(self) -> int:
        return int(self._lib.tfb_kernel_launches(self.handle))


def plan_kernels(k: int, sms: int = 148) -> list[tuple[int, int, int]]:
    """The kernel launches a fused bootstrap of k gates runs as: [(variant, gates per CTA, gates)], variant
    4 = K1d (one gate per warp), 5 = K1e (one gate per two-CTA cluster; gates per CTA reported as 0)."""
    v, w, g = (ctypes.c_int32 * 8)(), (ctypes.c_int32 * 8)(), (ctypes.c_int64 * 8)()
    n = lib().tfb_debug_plan_kernels(int(k), int(sms), v, w, g, 8)
    return [(int(v[i]), int(w[i]), int(g[i])) for i in range(n)]


def measure_peaks(device: int = 0) -> dict:
    d, i = ctypes.c_double(), ctypes.c_double()
    status = lib().tfb_measure_peaks(int(device), ctypes.byref(d), ctypes.byref(i))
    if status != 0:
        raise TfbError(f"tfb_measure_peaks failed with status {status}")
    return {"fp64_tflops": d.value, "int32_tops": i.value}
