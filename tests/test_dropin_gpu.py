"""Drop-in proof: the reference's OWN unit suite and acceptance program,
linked so that fassmvs::estimate_bundle, dog_mask and
geometric_consistency_mask are served by the B200 library through
include/fassmvs_b200.hpp (oracle/Makefile target `dropin`), pass on the GPU,
and the acceptance run prints exactly the golden numbers of
proj/test_output.txt:13-22 (the B200 path is bit-exact with the reference)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _binary(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle dropin)")
    return path


def test_reference_unit_suite_through_b200(b200):
    r = subprocess.run([_binary("unit_tests_b200")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m and int(m.group(3)) == 0, r.stdout


def test_reference_acceptance_through_b200(b200):
    r = subprocess.run([_binary("acceptance_b200"), "/nonexistent-cli"], capture_output=True,
                       text=True, timeout=900)
    out = r.stdout
    for crit in (1, 2, 3, 4, 5, 6, 7, 8, 10):
        assert f"[PASS] criterion {crit}:" in out, out
    assert "L1-rel 0.00500633 (< 0.01) over 100% of DoG-valid pixels" in out, out
    assert ("plane 9.22216 deg, sn 7.53061 deg, pg 7.44664 deg" in out
            and "L1-rel 0.00346314/0.00329057/0.00296517" in out), out
    assert "keeps 90.3847% of clean pixels" in out, out
