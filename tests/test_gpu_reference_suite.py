"""The reference's OWN test suite (chunkattn 0.1.0, pkg/tests, staged unmodified
in oracle/_ref/tests by oracle/make_ref.py) run against this package: the
plugin tests/refsuite_shim.py resolves ``chunkattn.attention / selection /
numerics / planner / reports`` to this package's GPU modules (the reference's
``rollout`` and ``cli`` run on top of them).

Every reference test must pass except the ones listed in EXPECTED, each for a
stated reason that is not an API or selection difference:

* fp64-precision assertions (atol 1e-5 against an fp64 token oracle, or an
  exact value copy): the kernels compute attention in bf16 with fp32
  accumulation by design (our tolerance rel-L2 1e-2);
* wall-clock shape assertions written for the CPU engine on toy sizes, where
  the GPU path's fixed host / launch overheads dominate (speedup >= 3 of a
  0.4 ms dense call; selection <= 10 % of a ~20 us kernel);
* the ``chunkattn`` console script, which only a pip install of the
  reference would put on PATH.
"""

from __future__ import annotations

import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "oracle", "_ref", "tests")

EXPECTED = {
    "test_acceptance.py::test_criterion_1_kernel_matches_token_oracle": "fp64 precision",
    "test_attention.py::test_dense_matches_oracle": "fp64 precision",
    "test_attention.py::test_dense_single_key_is_value_copy": "fp64 precision (bf16 copy)",
    "test_attention.py::test_sparse_matches_token_oracle": "fp64 precision",
    "test_attention.py::test_sparse_oracle_property": "fp64 precision",
    "test_acceptance.py::test_criterion_5_sparsity_proportional_cost": "wall-clock shape",
    "test_acceptance.py::test_criterion_8_selection_overhead_small": "wall-clock shape",
    "test_cli.py::test_console_script_installed": "console script not installed",
}


@pytest.mark.gpu
def test_reference_suite_against_this_package(tmp_path):
    if not os.path.isdir(SUITE):
        pytest.fail("reference suite not staged in oracle/_ref/tests (oracle/make_ref.py)")
    xml = tmp_path / "ref.xml"
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""),
               PYTHONDONTWRITEBYTECODE="1")
    proc = subprocess.run(
        [sys.executable, "-m", "pytest", "-p", "tests.refsuite_shim", SUITE, "-q",
         "-p", "no:cacheprovider", f"--junitxml={xml}"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    root = ET.parse(xml).getroot()
    passed, failed = [], []
    for case in root.iter("testcase"):
        name = f"{case.get('file', '').split('/')[-1] or case.get('classname').split('.')[-1] + '.py'}" \
               f"::{case.get('name')}"
        bad = case.find("failure") is not None or case.find("error") is not None
        skipped = case.find("skipped") is not None
        if bad:
            failed.append(name)
        elif not skipped:
            passed.append(name)
    unexpected = [n for n in failed if n not in EXPECTED]
    print(f"reference suite on the GPU package: {len(passed)} passed, {len(failed)} failed "
          f"({len(failed) - len(unexpected)} expected: "
          f"{sorted(set(EXPECTED[n] for n in failed if n in EXPECTED))})")
    assert not unexpected, f"unexpected failures: {unexpected}\n{proc.stdout[-3000:]}"
    assert len(passed) >= 150, (len(passed), proc.stdout[-2000:])
