"""Stage the real reference package into ``oracle/_ref/`` (TEST INFRASTRUCTURE).

The reference (``chunkattn`` 0.1.0, /root/reference/pkg/src/chunkattn) is
pure Python + NumPy (pyproject.toml:10-12): there is nothing to compile, so
"building" it is copying its eight source files, unmodified, into
``oracle/_ref/chunkattn/``.  ``oracle/_ref/`` is git-ignored (no reference
source enters the history) but not gpurun-ignored, so the staged copy travels
to the GPU box, where /root/reference does not exist.  Users:

  * tests/test_gpu_backends.py -- ``chunkattn.rollout()`` driving this
    package's backends, and the reference CPU rollout they are compared with;
  * bench.py's reference arm -- times the real ``hsa_attention`` at the
    aligned n = 1536 shape beside the framewise port (n = 1560 is rejected by
    the reference itself, selection.py:88-92);
  * tests/test_gpu_reference_suite.py -- the reference's own test suite
    (staged to ``oracle/_ref/tests/``) run against this package.

Never imported by ``paper_2602_04789_b200/``.

    python oracle/make_ref.py            # no-op when /root/reference is absent
"""

from __future__ import annotations

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = "/root/reference/pkg/src/chunkattn"
DST = os.path.join(HERE, "_ref", "chunkattn")


TESTS_SRC = "/root/reference/pkg/tests"
TESTS_DST = os.path.join(HERE, "_ref", "tests")


def stage(src: str = SRC, dst: str = DST) -> str | None:
    """Copy the reference package and its test suite (tests/test_gpu_reference_suite.py
    runs that suite against this package); returns the _ref directory (None if no
    source)."""
    if not os.path.isdir(src):
        return os.path.dirname(dst) if os.path.isdir(dst) else None
    os.makedirs(dst, exist_ok=True)
    for name in sorted(os.listdir(src)):
        if name.endswith(".py"):
            shutil.copyfile(os.path.join(src, name), os.path.join(dst, name))
    if os.path.isdir(TESTS_SRC):
        os.makedirs(TESTS_DST, exist_ok=True)
        for name in sorted(os.listdir(TESTS_SRC)):
            if name.endswith(".py"):
                shutil.copyfile(os.path.join(TESTS_SRC, name), os.path.join(TESTS_DST, name))
    with open(os.path.join(os.path.dirname(dst), "SOURCE"), "w") as fh:
        fh.write(f"{src}\n")
    return os.path.dirname(dst)


def ref_path() -> str | None:
    """Directory to put on sys.path to import the staged ``chunkattn`` (None if not staged)."""
    d = os.path.dirname(DST)
    return d if os.path.isfile(os.path.join(DST, "__init__.py")) else None


def import_reference():
    """Import the staged reference package (raises ImportError when not staged)."""
    d = ref_path()
    if d is None:
        raise ImportError("oracle/_ref/chunkattn is not staged (run python oracle/make_ref.py "
                          "where /root/reference exists)")
    if d not in sys.path:
        sys.path.insert(0, d)
    sys.dont_write_bytecode = True
    import chunkattn  # noqa: PLC0415
    if not os.path.abspath(chunkattn.__file__).startswith(os.path.abspath(d)):
        raise ImportError(f"chunkattn resolved to {chunkattn.__file__}, not the staged copy")
    return chunkattn


if __name__ == "__main__":
    print(stage())
