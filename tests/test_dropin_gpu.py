"""Drop-in proof: the reference's OWN unit suite and acceptance program,
linked so that fassmvs::estimate_bundle, every stage-level function of the
reference API (build_pyramids, gaussian_blur, upscale_nearest, refine_range,
median_filter_5x5, census_transform, sweep_cost_volume, aggregate,
aggregate_single_path, wta, compute_normal_offsets, normals_from_depth,
smooth_normals, confidence_map, the host geometry), the post-filters and the
CLI's output stage (colorize_*, write_pfm, write_png; test_io.cpp:32-66,168-181,
240-270) are
served by the B200 library through include/fassmvs_b200.hpp (oracle/Makefile
target `dropin`), pass on the GPU, and the acceptance run prints exactly the
golden numbers of proj/test_output.txt:13-22 (the B200 path is bit-exact with
the reference). The reference's own independent oracles (test_sgm.cpp:157-200
exhaustive labelings and chain DP in all 8 directions, test_matching.cpp:26-69
census known answers, acceptance.cpp:131-153 criterion 1's 200 random volumes
vs chain_dp) thereby check the GPU kernels."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _binary(name):
    path = os.path.join(REF_DIR, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle dropin)")
    return path


# symbols the drop-in binaries must take from the drop-in TU (which calls the
# C ABI of libfmvs.so), never from the reference's CPU sources
DROPIN_SYMBOLS = ["estimate_bundle", "build_pyramids", "gaussian_blur", "upscale_nearest", "refine_range",
                  "median_filter_5x5", "census_transform", "sweep_cost_volume", "aggregate",
                  "aggregate_single_path", "wta", "compute_normal_offsets", "normals_from_depth",
                  "smooth_normals", "confidence_map", "plane_distances", "plane_homography", "dog_mask",
                  "geometric_consistency_mask", "colorize_depth", "colorize_normals", "colorize_confidence",
                  "write_pfm", "write_png"]
C_ABI = ["fmvs_estimate_bundle", "fmvs_build_pyramids", "fmvs_sweep_cost_volume", "fmvs_aggregate",
         "fmvs_aggregate_single_path", "fmvs_wta", "fmvs_compute_normal_offsets", "fmvs_median_filter_5x5",
         "fmvs_normals_from_depth", "fmvs_smooth_normals", "fmvs_confidence_map", "fmvs_refine_range",
         "fmvs_upscale_nearest", "fmvs_gaussian_blur", "fmvs_census_transform", "fmvs_plane_distances",
         "fmvs_colorize_depth", "fmvs_colorize_normals", "fmvs_colorize_confidence", "fmvs_write_pfm",
         "fmvs_write_png"]


@pytest.mark.parametrize("name", ["unit_tests_b200", "acceptance_b200"])
def test_dropin_symbols_resolve_into_libfmvs(name):
    """nm: each drop-in symbol is defined once (the drop-in TU), the CPU
    definitions exist only under their renamed *_cpu names, and the C ABI
    entry points they call are undefined in the binary (resolved from
    libfmvs.so, which ldd shows the binary loads)."""
    path = _binary(name)
    nm = subprocess.run(["nm", "-C", path], capture_output=True, text=True, check=True).stdout
    defined = {}
    undefined = set()
    for ln in nm.splitlines():
        parts = ln.split(None, 2)
        if len(parts) == 3 and parts[1] in ("T", "W"):
            nm_name = parts[2].split("(")[0]
            defined[nm_name] = defined.get(nm_name, 0) + 1
        elif len(parts) == 2 and parts[0] == "U":
            undefined.add(parts[1])
    for sym in DROPIN_SYMBOLS:
        assert f"fassmvs::{sym}_cpu" in defined or sym in ("dog_mask", "geometric_consistency_mask"), sym
    for entry in C_ABI:
        assert entry in undefined, entry
    ldd = subprocess.run(["ldd", path], capture_output=True, text=True, check=True).stdout
    assert "libfmvs.so" in ldd


@pytest.mark.gpu
def test_reference_unit_suite_through_b200(b200):
    r = subprocess.run([_binary("unit_tests_b200")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed", r.stdout)
    assert m and int(m.group(3)) == 0, r.stdout


@pytest.mark.gpu
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
