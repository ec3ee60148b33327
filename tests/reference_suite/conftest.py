"""Run the reference's own unit tests against the drop-in.

tests/reference_suite/_ref/ holds unmodified copies of
/root/reference/pkg/tests/{test_charts,test_geometry,test_packing,
test_metrics,test_baselines}.py plus their conftest.py / oracles.py, made by
sync_reference_tests.py in the build container (git-ignored; it travels to
the GPU box with the snapshot).  Here `atlaspack` -- the module name those
files import -- is aliased onto paper_2502_17712_b200, so each reference
test calls the CUDA path through the reference's own API.  Every collected
reference test is marked `gpu` (the compute calls need a B200).

Out of scope, and so expected to fail: the tiny-instance brute-force test
oracle `exhaustive_optimal` (baselines.py:272-318), which is not part of the
per-frame path.
"""

import importlib
import os
import sys
import types

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

# test node-id fragments -> reason (xfail, strict: a pass would mean the list is stale)
OUT_OF_SCOPE = {
    "test_baselines.py::TestExhaustiveOptimal": "exhaustive_optimal (baselines.py:272-318) is out of scope",
}


def _install_alias():
    if "atlaspack" in sys.modules and getattr(sys.modules["atlaspack"], "__drop_in__", False):
        return
    import paper_2502_17712_b200 as pkg
    alias = types.ModuleType("atlaspack")
    alias.__dict__.update({k: getattr(pkg, k) for k in dir(pkg) if not k.startswith("__")})
    alias.__path__ = []
    alias.__drop_in__ = True

    def exhaustive_optimal(*args, **kwargs):
        raise NotImplementedError("exhaustive_optimal is out of scope for the drop-in")

    alias.exhaustive_optimal = exhaustive_optimal
    sys.modules["atlaspack"] = alias
    for sub in ("charts", "geometry", "packing", "metrics", "baselines", "cli"):
        mod = importlib.import_module(f"paper_2502_17712_b200.{sub}")
        sys.modules[f"atlaspack.{sub}"] = mod
        setattr(alias, sub, mod)


if os.path.isdir(REF_DIR):
    _install_alias()
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)  # the reference tests' `from oracles import ...`


def pytest_collection_modifyitems(config, items):
    for item in items:
        path = str(item.fspath)
        if not path.startswith(REF_DIR + os.sep):
            continue
        item.add_marker(pytest.mark.gpu)
        for frag, why in OUT_OF_SCOPE.items():
            if frag in item.nodeid:
                item.add_marker(pytest.mark.xfail(reason=why, raises=NotImplementedError, strict=True))
