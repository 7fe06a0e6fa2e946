"""The remaining public helpers of the reference API (matching.hpp,
geometry.hpp, pipeline.hpp) against the oracle: host helpers bit for bit on
the CPU (census_bits_at, ncc_cost incl. the known answers of
test_matching.cpp:77-102, apply_homography, cross_ratio,
require_centers_in_front), device helpers (census_transform, gaussian_blur)
bit for bit on the GPU."""
import numpy as np
import pytest

from paper_2112_00821_b200 import ConfigError, GeometryError, InvalidInputError


def test_census_bits_at(b200_host, oracle):
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, (13, 17)).astype(np.uint8)
    for x, y in [(0, 0), (16, 12), (5, 6), (0, 12), (16, 0)]:
        for ww, wh in [(5, 5), (9, 7), (3, 3)]:
            assert b200_host.census_bits_at(img, x, y, ww, wh) == oracle.census_bits_at(img, x, y, ww, wh)


def test_ncc_cost_known_answers_and_parity(b200_host, oracle):
    rng = np.random.default_rng(4)
    a = rng.uniform(0, 255, 25).astype(np.float32)
    for be in (b200_host, oracle):
        assert be.ncc_cost(a, a) == 0                           # identical
        assert be.ncc_cost(a, 2.0 * a + 7.0) == 0               # affine
        assert be.ncc_cost(a, -a) == 255                        # negated
        assert be.ncc_cost(a, np.full(25, 9.0, np.float32)) == 255  # flat
        with pytest.raises(InvalidInputError):
            be.ncc_cost(a, a[:5])
    for _ in range(50):
        b = (a + rng.normal(0, 40, 25)).astype(np.float32)
        assert b200_host.ncc_cost(a, b) == oracle.ncc_cost(a, b)


def test_apply_homography_and_cross_ratio(b200_host, oracle):
    rng = np.random.default_rng(5)
    for _ in range(20):
        h = rng.normal(size=(3, 3))
        h[2, 2] += 3.0
        x, y = rng.uniform(-50, 50, 2)
        assert np.array_equal(b200_host.apply_homography(h, x, y), oracle.apply_homography(h, x, y))
    for dims in (2, 3):
        p = rng.normal(size=(4, dims))
        assert b200_host.cross_ratio(*p) == oracle.cross_ratio(*p)
        with pytest.raises(InvalidInputError):
            b200_host.cross_ratio(p[0], p[1], p[1], p[0])
        with pytest.raises(InvalidInputError):
            oracle.cross_ratio(p[0], p[1], p[1], p[0])


def test_require_centers_in_front(b200_host, oracle):
    n = (0.0, 0.0, -1.0)
    ok = [[0.0, 0.0, 0.0], [1.0, 0.5, -2.0]]
    bad = ok + [[0.0, 0.0, 6.0]]
    for be in (b200_host, oracle):
        be.require_centers_in_front(n, 5.0, ok)
        with pytest.raises(GeometryError):
            be.require_centers_in_front(n, 5.0, bad)


@pytest.mark.gpu
def test_census_transform_and_blur_bitexact(b200, oracle):
    rng = np.random.default_rng(6)
    img = rng.integers(0, 256, (29, 41)).astype(np.uint8)
    for ww, wh in [(5, 5), (9, 7), (1, 1), (7, 9)]:
        assert np.array_equal(b200.census_transform(img, ww, wh), oracle.census_transform(img, ww, wh))
    for be in (b200, oracle):
        with pytest.raises(ConfigError):
            be.census_transform(img, 4, 5)
        with pytest.raises(ConfigError):
            be.census_transform(img, 9, 9)
    for radius, sigma in [(1, 1.0), (3, 1.4), (2, 0.7), (0, 1.0)]:
        assert np.array_equal(b200.gaussian_blur(img, radius, sigma), oracle.gaussian_blur(img, radius, sigma))
    one = img[:1, :1].copy()
    assert np.array_equal(b200.gaussian_blur(one, 3, 1.4), oracle.gaussian_blur(one, 3, 1.4))
