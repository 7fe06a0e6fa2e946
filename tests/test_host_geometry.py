"""Host-side geometry of the B200 library vs the oracle, bit for bit, on CPU.

Every sweep sample depends on the homographies and every plane interval on
the plane stack, so these must be bit-identical, not just close
(SURVEY.md Appendix A). Error types must match too."""
import numpy as np
import pytest

from paper_2112_00821_b200 import GeometryError, Intrinsics, InvalidInputError, Pose

from scenes import random_camera_pair


def test_plane_homography_bitexact(b200_host, oracle, rng):
    for _ in range(200):
        k, ref, other = random_camera_pair(rng)
        n = np.array([rng.uniform(-0.2, 0.2), rng.uniform(-0.2, 0.2), -1.0])
        n /= np.linalg.norm(n)
        d = float(rng.uniform(1, 50))
        a = b200_host.plane_homography(n, d, k, ref, k, other)
        b = oracle.plane_homography(n, d, k, ref, k, other)
        assert np.array_equal(a, b)


def test_bounding_distances_bitexact(b200_host, oracle, rng):
    for _ in range(100):
        k, _, _ = random_camera_pair(rng)
        n = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), -1.0])
        n /= np.linalg.norm(n)
        lo, hi = sorted(rng.uniform(1, 60, 2))
        assert b200_host.bounding_distances(lo, hi, n, k) == oracle.bounding_distances(lo, hi, n, k)


@pytest.mark.parametrize("max_planes", [2, 7, 64, 100000])
def test_plane_distances_bitexact(b200_host, oracle, rng, max_planes):
    for _ in range(60):
        k, ref, other = random_camera_pair(rng)
        n = np.array([0.0, rng.uniform(-0.4, 0.4), -1.0])
        n /= np.linalg.norm(n)
        lo, hi = sorted(rng.uniform(2, 40, 2))
        try:
            dlo, dhi = oracle.bounding_distances(lo, hi, n, k)
            want = oracle.plane_distances(k, ref, k, other, dlo, dhi, n, max_planes)
        except GeometryError:
            with pytest.raises(GeometryError):
                dlo, dhi = b200_host.bounding_distances(lo, hi, n, k)
                b200_host.plane_distances(k, ref, k, other, dlo, dhi, n, max_planes)
            continue
        got = b200_host.plane_distances(k, ref, k, other, dlo, dhi, n, max_planes)
        assert np.array_equal(got, want)


def test_plane_distances_errors_match(b200_host, oracle):
    k = Intrinsics(100.0, 100.0, 31.5, 23.5, 64, 48)
    ref = Pose()
    same = Pose()
    for be in (b200_host, oracle):
        with pytest.raises(GeometryError):  # zero baseline
            be.plane_distances(k, ref, k, same, 5.0, 10.0, (0, 0, -1), 64)
        with pytest.raises(InvalidInputError):
            be.plane_distances(k, ref, k, same, -1.0, 10.0, (0, 0, -1), 64)
        assert list(be.plane_distances(k, ref, k, same, 5.0, 5.0, (0, 0, -1), 64)) == [5.0]


def test_depth_from_plane_and_scalars(b200_host, oracle, rng):
    k = Intrinsics(120.0, 110.0, 40.2, 30.7, 80, 60)
    for _ in range(200):
        x, y = rng.uniform(-5, 85), rng.uniform(-5, 65)
        n = rng.uniform(-1, 1, 3)
        n /= np.linalg.norm(n)
        d = float(rng.uniform(0.5, 30))
        assert b200_host.depth_from_plane(x, y, n, d, k) == oracle.depth_from_plane(x, y, n, d, k)
    for di in range(256):
        assert b200_host.adaptive_phi2(100.0, 8.0, 10.0, di) == oracle.adaptive_phi2(100.0, 8.0, 10.0, di)
    assert oracle.adaptive_phi2(100.0, 8.0, 10.0, 0.0) == 900.0  # test_sgm.cpp:136
    for _ in range(200):
        a, b, c = sorted(rng.uniform(1, 20, 3))
        cs = rng.uniform(0, 1000, 3)
        if not (a < b < c):
            continue
        assert b200_host.parabola_refine(a, b, c, *cs) == oracle.parabola_refine(a, b, c, *cs)
    for be in (b200_host, oracle):
        with pytest.raises(InvalidInputError):
            be.parabola_refine(3.0, 2.0, 4.0, 1, 0, 1)
