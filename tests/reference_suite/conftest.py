"""Run the reference's own test suite (/root/reference/pkg/tests, 189 tests)
against this package, imported under the reference's name ``hjls``.

The test files are NOT committed (they are the reference's source):
``python scripts/stage_reference_suite.py`` copies them into
``tests/reference_suite/_staged/`` (git-ignored; it travels to the GPU box
with the gpurun snapshot) and ``HJ_REFERENCE_SUITE=1 python -m pytest
tests/reference_suite -m gpu`` runs them there.  Without that variable this
directory collects nothing, so the default test runs are unaffected.

Every staged test is marked ``gpu``: the package has no CPU path.  The one
test excluded is the reference's own documented known-red
``test_rockets_brt_desk_scale`` (pkg/tests/test_acceptance.py:6-14, 210-244:
red on the reference itself).
"""
import importlib
import os
import sys

import pytest

STAGED = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_staged")
ENABLED = os.environ.get("HJ_REFERENCE_SUITE") == "1" and os.path.isdir(STAGED)
KNOWN_RED = {"test_rockets_brt_desk_scale": "known-red on the reference itself (test_acceptance.py:6-14)"}
SUBMODULES = ("grid", "shapes", "spatial", "term", "integrator", "reachability", "snapshot", "cli", "selftest")

if not ENABLED:
    collect_ignore_glob = ["_staged/*", "_staged"]
else:
    import paper_2411_03501_b200 as _pkg

    sys.modules["hjls"] = _pkg
    for _name in SUBMODULES:
        sys.modules[f"hjls.{_name}"] = importlib.import_module(f"paper_2411_03501_b200.{_name}")


def pytest_collection_modifyitems(config, items):
    for item in items:
        if STAGED not in str(item.fspath):
            continue
        item.add_marker(pytest.mark.gpu)
        if item.originalname in KNOWN_RED or item.name in KNOWN_RED:
            item.add_marker(pytest.mark.skip(reason=KNOWN_RED.get(item.originalname, "known red")))
