"""INTEGRATION.md §1's maintainer-side binding compiled against the reference.

oracle/_ref/binding_check is include/lamina_b200_binding.hpp (lamina::copyViewB200) built
against the reference's own headers and objects and this repo's C ABI library (oracle/Makefile
target `binding`).  It runs lamina::copyView and lamina::copyViewB200 on the same
lamina::View objects over 100+ layout pairs (instrumented ones included) and compares every
blob byte and every counter, plus the "incompatible views" and user-defined-mapping errors.
"""
import os
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "oracle", "_ref", "binding_check")


def test_copy_view_b200_binding_matches_reference_copy_view():
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/binding_check not built (make -C oracle binding)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    tail = "\n".join(r.stdout.strip().splitlines()[-5:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "binding_check: OK" in tail, tail
