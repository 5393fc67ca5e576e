"""The reference's own doctest unit suites for the hot-path modules (proj/tests/test_{engine,
retrieval,maintainer,index,store,harness}.cpp), compiled unmodified against the C++ drop-in
(include/kvclust_b200*.hpp -> libkvclust_b200.so -> libkvc.so; tests/cpp/Makefile, `unit_b200`)
and run on the GPU: every case the reference library passes (`unit_ref`, 70 cases on the CPU) must
pass through the GPU engine. doctest itself is absent from the image; tests/cpp/doctest_shim
stands in for it (same macros, one [PASS]/[FAIL] line per case)."""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "_build", "unit_b200")


def test_reference_unit_suites_on_the_dropin():
    if not os.path.exists(BIN):
        pytest.skip("tests/cpp/_build/unit_b200 not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=1500, cwd=os.path.dirname(BIN))
    print(r.stdout[-6000:])
    print(r.stderr[-3000:])
    failed = [ln for ln in r.stdout.splitlines() if ln.startswith("[FAIL]")]
    m = re.search(r"cases: (\d+) failed: (\d+)", r.stdout)
    assert m, r.stdout[-2000:]
    assert int(m.group(1)) == 70, m.group(0)
    assert failed == [] and int(m.group(2)) == 0, failed
    assert r.returncode == 0
