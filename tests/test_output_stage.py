"""Output stage of the CLI: PFM writer (map_io.cpp:34-44,
95-113) and the colorize visualisations (colorize.cpp:32-70), byte for byte
against the reference. The PFM writer is host code (CPU test); colorize runs
on the device (gpu)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT

PFM_TOOL = os.path.join(ROOT, "oracle", "_ref", "pfm_tool")


@pytest.mark.parametrize("shape", [(7, 5), (6, 4, 3), (1, 1), (1, 9, 3)])
def test_write_pfm_bytes_match_reference(b200_host, oracle, tmp_path, shape):
    if not os.path.exists(PFM_TOOL):
        pytest.skip("oracle pfm_tool not built")
    rng = np.random.default_rng(len(shape) * 100 + shape[0])
    data = rng.normal(size=shape).astype(np.float32)
    data.flat[0] = np.nan
    a, b = tmp_path / "b200.pfm", tmp_path / "ref.pfm"
    b200_host.write_pfm(str(a), data)
    ch = 1 if len(shape) == 2 else 3
    subprocess.run([PFM_TOOL, str(b), str(shape[1]), str(shape[0]), str(ch)], input=data.tobytes(),
                   check=True)
    assert a.read_bytes() == b.read_bytes()
    hdr = b"Pf\n" if len(shape) == 2 else b"PF\n"
    assert a.read_bytes().startswith(hdr)


def test_write_pfm_error(b200_host):
    from paper_2112_00821_b200 import InvalidInputError
    with pytest.raises(InvalidInputError):
        b200_host.write_pfm("/nonexistent-dir/x.pfm", np.zeros((2, 2), np.float32))


@pytest.mark.gpu
def test_colorize_bitexact(b200, oracle):
    rng = np.random.default_rng(7)
    h, w = 37, 53
    d = rng.uniform(2.0, 45.0, (h, w)).astype(np.float32)
    d[rng.random((h, w)) < 0.1] = 0.0
    d[0, :5] = [np.nan, np.inf, -1.0, 4.0, 40.0]
    for lo, hi in [(4.0, 40.0), (10.0, 10.0), (40.0, 4.0), (0.0, 1e-3)]:
        assert np.array_equal(b200.colorize_depth(d, lo, hi), oracle.colorize_depth(d, lo, hi)), (lo, hi)
    n = rng.normal(size=(h, w, 3)).astype(np.float32) * 0.8
    n[rng.random((h, w)) < 0.1] = 0.0
    n[1, :3] = [[2.0, -3.0, 0.5], [1.0, 1.0, 1.0], [-1.0, -1.0, -1.0]]
    assert np.array_equal(b200.colorize_normals(n), oracle.colorize_normals(n))
    c = rng.uniform(-0.5, 1.5, (h, w)).astype(np.float32)
    c[2, :4] = [0.0, 1.0, 0.5, 0.001960784]
    assert np.array_equal(b200.colorize_confidence(c), oracle.colorize_confidence(c))
