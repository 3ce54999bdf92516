"""pytest plugin (test infrastructure): run the REFERENCE's own test suite
against this package.

    python -m pytest -p tests.refsuite_shim oracle/_ref/tests

The staged, unmodified reference tests (oracle/make_ref.py) import
``chunkattn.attention``, ``.selection``, ``.numerics``, ``.planner`` and
``.reports``; this plugin makes those names resolve to this package's modules
(the GPU hot path), so the reference's assertions run on the sm_100a kernels.
``chunkattn.rollout`` and ``chunkattn.cli`` (outside the hot path)
stay the reference's own files, executed on top of the substituted modules --
their HsaBackend / bench / mask-dump therefore call the GPU kernels too.
"""

from __future__ import annotations

import importlib.util
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref", "chunkattn")


def install() -> None:
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    from paper_2602_04789_b200 import attention, numerics, planner, reports, selection
    pkg = types.ModuleType("chunkattn")
    pkg.__path__ = [REF]
    pkg.__file__ = os.path.join(REF, "__init__.py")
    sys.modules["chunkattn"] = pkg
    for name, mod in (("attention", attention), ("selection", selection),
                      ("numerics", numerics), ("planner", planner), ("reports", reports)):
        sys.modules[f"chunkattn.{name}"] = mod
        setattr(pkg, name, mod)
    for name in ("rollout", "cli"):
        spec = importlib.util.spec_from_file_location(f"chunkattn.{name}",
                                                      os.path.join(REF, f"{name}.py"))
        mod = importlib.util.module_from_spec(spec)
        sys.modules[f"chunkattn.{name}"] = mod
        spec.loader.exec_module(mod)
        setattr(pkg, name, mod)


def pytest_configure(config):
    sys.dont_write_bytecode = True
    install()
