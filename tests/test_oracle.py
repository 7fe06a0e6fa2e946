"""Pins the parity oracle before anything is compared against it (CPU only).

1. The reference's own unit suite (proj/tests/test_*.cpp, 104 doctest cases)
   passes when built against the Eigen shim.
2. The reference's acceptance run reproduces the golden numbers recorded with
   real Eigen in proj/test_output.txt:13-22 to every printed digit.
3. The independent numpy restatement (oracle/restate.py) agrees with the
   oracle bit for bit on random ragged volumes (SGM, WTA) and maps (median).
4. The oracle reproduces the committed golden fixtures (tests/golden/).
"""
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

sys.path.insert(0, os.path.join(ROOT, "oracle"))
import restate  # noqa: E402

from paper_2112_00821_b200 import CostVolume, Intrinsics, PlaneStack, SgmConfig, SgmVariant  # noqa: E402
from scenes import harmonic_stack, random_volume  # noqa: E402

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _binary(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle tests)")
    return path


def test_reference_unit_suite_passes_under_the_shim(oracle):
    r = subprocess.run([_binary("unit_tests")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m and int(m.group(1)) == 104 and int(m.group(3)) == 0, r.stdout


def test_acceptance_golden_numbers_reproduce(oracle):
    """test_output.txt:13-22 (real Eigen) vs the shim-built oracle."""
    r = subprocess.run([_binary("acceptance"), "/nonexistent-cli"], capture_output=True, text=True,
                       timeout=900)
    out = r.stdout
    for crit in (1, 2, 3, 4, 5, 6, 7, 8, 10):
        assert f"[PASS] criterion {crit}:" in out, out
    assert "L1-rel 0.00500633 (< 0.01) over 100% of DoG-valid pixels" in out
    assert ("plane 9.22216 deg, sn 7.53061 deg, pg 7.44664 deg" in out
            and "L1-rel 0.00346314/0.00329057/0.00296517" in out), out
    assert "keeps 90.3847% of clean pixels" in out
    assert "phi2(0) = 900 (exactly 900)" in out
    # criterion 9 needs the reference CLI (CLI11 is not vendored): out of scope


@pytest.mark.parametrize("adaptive", [False, True])
def test_restated_sgm_matches_oracle(oracle, adaptive):
    rng = np.random.default_rng(7)
    intr = Intrinsics(100.0, 100.0, 4.5, 3.0, 10, 7)
    for trial in range(3):
        w, h, planes = 10, 7, 9
        first, count, offset, costs = random_volume(rng, w, h, planes)
        img = rng.integers(0, 256, (h, w)).astype(np.uint8)
        vol = CostVolume(w, h, PlaneStack(harmonic_stack(planes)), 2, first, count, offset, costs)
        cfg = SgmConfig(SgmVariant.Plane, 8, 7.0, adaptive, 40.0, 8.0, 10.0, 2)
        for dx, dy in [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1), (1, -1), (-1, 1)]:
            want = oracle.aggregate_single_path(vol, img, cfg, intr, dx, dy).values
            got = restate.sgm_single_path(first, count, offset, costs, img, w, h, dx, dy, cfg.phi1,
                                          cfg.phi2_fixed, cfg.phi2_adaptive, cfg.alpha, cfg.beta,
                                          cfg.penalty_scale)
            assert np.array_equal(got, want), (trial, dx, dy)


def test_restated_wta_and_median_match_oracle(oracle):
    rng = np.random.default_rng(3)
    w, h = 23, 17
    first, count, offset, _ = random_volume(rng, w, h, 12)
    values = rng.integers(0, 50, int(count.sum())).astype(np.uint32)  # many ties
    from paper_2112_00821_b200 import AggregatedVolume
    agg = AggregatedVolume(w, h, PlaneStack(harmonic_stack(12)), first, count, offset, values)
    assert np.array_equal(restate.wta(first, count, offset, values, w, h), oracle.wta(agg))
    depth = rng.uniform(1, 5, (h, w)).astype(np.float32)
    depth[rng.random((h, w)) < 0.3] = 0.0
    assert np.array_equal(restate.median_5x5(depth), oracle.median_filter_5x5(depth))


def test_restated_census_cost_matches_lut():
    # matching.cpp:249-260 on hand-made windows: identical -> 0, reversed -> 255
    win = np.arange(25, dtype=np.float64)
    bits = 0
    for i, v in enumerate(win):
        if i == 12:
            continue
        bits = (bits << 1) | (1 if v < win[12] else 0)
    assert restate.census_cost(win, bits, 24) == 0
    assert restate.census_cost(win, bits ^ ((1 << 24) - 1), 24) == 255
    assert restate.census_cost(np.full(25, 3.0), 0, 24) == 0


GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("name", ["smoke", "c4_fronto_ncc", "census_sn_3lvl"])
def test_oracle_reproduces_golden_fixtures(oracle, name):
    sys.path.insert(0, GOLDEN)
    import make_golden
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    bundle, cfg = make_golden.case(oracle, name)
    r = oracle.estimate_bundle(bundle, cfg)
    assert np.array_equal(r.depth, g["depth"])
    assert np.array_equal(r.normals, g["normals"])
    assert np.array_equal(r.confidence, g["confidence"])
