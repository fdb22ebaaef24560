"""pytest plugin (test infrastructure): run the REFERENCE's own test files
(baseline/_ref/ref_tests, copied from /root/reference/pkg/tests by
__graft_entry__.build()) against the unmodified reference package with the B200
backend registered through ``paper_1511_07207_b200.plugin.install``.

Every backend object a reference test builds -- the ``backend`` fixture of its
conftest.py (reference / blocked) and direct ``ReferenceBackend()`` /
``BlockedBackend()`` constructions -- is replaced by the registered B200 backend,
so the reference solvers dispatch to the device path.

DENSOLVE_REF_SUITE_MODE=fused (default): solver calls run this package's fused
device solvers; =ops: the reference's own solver loops run over the B200 op contract.
"""
import os
import sys

import pytest

MODE = os.environ.get("DENSOLVE_REF_SUITE_MODE", "fused")
_REF_TESTS = os.path.realpath(os.environ.get("DENSOLVE_REF_TESTS", ""))


def pytest_configure(config):
    import densolve

    from paper_1511_07207_b200 import plugin
    plugin.install(densolve, fused=(MODE == "fused"))


def _ref_test_modules():
    for mod in list(sys.modules.values()):
        f = getattr(mod, "__file__", None) or ""
        if f and os.path.realpath(f).startswith(_REF_TESTS + os.sep):
            yield mod


@pytest.fixture(autouse=True)
def _b200_everywhere(monkeypatch):
    import densolve

    from paper_1511_07207_b200 import plugin
    cls = densolve._b200_plugin

    def make(*_a, **_k):
        return cls()

    for mod in _ref_test_modules():
        plugin.rebind_module(densolve, mod)
        for name in ("ReferenceBackend", "BlockedBackend"):
            if hasattr(mod, name):
                monkeypatch.setattr(mod, name, make)
    yield
