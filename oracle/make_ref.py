"""Stage the UNMODIFIED reference under oracle/_ref/ (git-ignored, travels to the GPU box).

TEST INFRASTRUCTURE.  The reference (`/root/reference/pkg`: pure Python + numpy, no build step) only
exists in the build container; the GPU box gets whatever sits in the repo snapshot.  This recipe copies
the reference's package sources and its own test-suite, byte for byte, to

    oracle/_ref/src/encirc/     <- /root/reference/pkg/src/encirc/
    oracle/_ref/tests/          <- /root/reference/pkg/tests/

so that (i) `tests/test_reference_suite.py` can run the reference's OWN tests with its
`OracleBootstrapEngine` replaced by the B200 binding, and (ii) `bench.py --impl reference` / the
`cpu_baseline` legs time the real reference instead of a port.  Nothing under `paper_2005_01945_b200/`
imports from here; nothing from here is committed (`.gitignore` lists oracle/_ref/).

    python oracle/make_ref.py [--source /root/reference/pkg]
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
DEST = os.path.join(HERE, "_ref")
DEFAULT_SOURCE = "/root/reference/pkg"


def stage(source: str = DEFAULT_SOURCE, dest: str = DEST) -> dict | None:
    """Copy the reference; returns the manifest, or None when the reference is not on this machine."""
    src_pkg, src_tests = os.path.join(source, "src", "encirc"), os.path.join(source, "tests")
    if not (os.path.isdir(src_pkg) and os.path.isdir(src_tests)):
        return None
    if os.path.isdir(dest):
        shutil.rmtree(dest)
    ignore = shutil.ignore_patterns("__pycache__", "*.pyc", ".pytest_cache", ".hypothesis")
    shutil.copytree(src_pkg, os.path.join(dest, "src", "encirc"), ignore=ignore)
    shutil.copytree(src_tests, os.path.join(dest, "tests"), ignore=ignore)
    manifest = {"source": source, "files": {}}
    for root, _, files in os.walk(dest):
        for name in sorted(files):
            path = os.path.join(root, name)
            with open(path, "rb") as fh:
                manifest["files"][os.path.relpath(path, dest)] = hashlib.sha256(fh.read()).hexdigest()
    with open(os.path.join(dest, "MANIFEST.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    return manifest


def available(dest: str = DEST) -> bool:
    return os.path.isfile(os.path.join(dest, "src", "encirc", "__init__.py"))


def import_reference(dest: str = DEST):
    """Import the staged reference package (`encirc`) and return the module."""
    if not available(dest):
        raise ImportError("oracle/_ref is not staged: run `python oracle/make_ref.py` where /root/reference exists")
    src = os.path.join(dest, "src")
    if src not in sys.path:
        sys.path.insert(0, src)
    import encirc

    return encirc


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--source", default=DEFAULT_SOURCE)
    got = stage(ap.parse_args().source)
    print("reference not found; nothing staged" if got is None else f"staged {len(got['files'])} files under {DEST}")
