"""pytest plugin (`-p tests.ref_b200_plugin`) that runs the REFERENCE's own test-suite against the B200
engine.  TEST INFRASTRUCTURE: it imports the staged reference (oracle/_ref, see oracle/make_ref.py).

Loaded before the reference's conftest.py and test modules are imported, it replaces
`encirc.OracleBootstrapEngine` by the binding of paper_2005_01945_b200.encirc_binding, so the reference's
`orc` / `engines` fixtures (pkg/tests/conftest.py:21-28) and every test that constructs
`OracleBootstrapEngine(key, seed, pool)` directly get a real-bootstrap GPU engine.

REF_BACKEND=host swaps the GPU for the C oracle behind the same binding (CPU smoke of the plumbing).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle.make_ref import import_reference  # noqa: E402

encirc = import_reference()

from paper_2005_01945_b200.encirc_binding import bind  # noqa: E402

_backend = None
if os.environ.get("REF_BACKEND") == "host":
    from tests.host_engine import HostOracleEngine

    def _backend(key, seed):
        return HostOracleEngine(key, seed, lazy=True)

STOCK = encirc.OracleBootstrapEngine
BOUND = bind(encirc, backend=_backend)
encirc.OracleBootstrapEngine = BOUND
encirc.engine.OracleBootstrapEngine = BOUND
for _name in ("bench", "cli"):  # modules that captured the name at import time
    _mod = sys.modules.get(f"encirc.{_name}")
    if _mod is not None and getattr(_mod, "OracleBootstrapEngine", None) is STOCK:
        _mod.OracleBootstrapEngine = BOUND


def pytest_report_header(config):
    return f"encirc.OracleBootstrapEngine -> {BOUND.__module__}.{BOUND.__qualname__} (backend: {os.environ.get('REF_BACKEND', 'b200')})"
