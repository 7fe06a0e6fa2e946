"""The median-of-25 selection network of the median filter kernel
(csrc/k_pixel.cu kMed25A/kMed25B, median_filter_5x5 of pipeline.cpp:175-198
when the whole 5x5 window is valid): element 12 after the network equals the
13th smallest value, for random, tied and constant windows (0-1 principle
checked on random binary inputs too). CPU only."""
import os
import re

import numpy as np

SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                   "paper_2112_00821_b200", "csrc", "k_pixel.cu")


def _network(name_a, name_b):
    s = open(SRC).read()
    a = [int(v) for v in re.search(name_a + r"\[[^\]]*\] = \{([^}]*)\}", s).group(1).split(",")]
    b = [int(v) for v in re.search(name_b + r"\[[^\]]*\] = \{([^}]*)\}", s).group(1).split(",")]
    return list(zip(a, b))


def _run(net, v):
    v = v.copy()
    for a, b in net:
        lo = np.minimum(v[:, a], v[:, b])
        hi = np.maximum(v[:, a], v[:, b])
        v[:, a], v[:, b] = lo, hi
    return v


def test_median25_network_selects_element_12():
    net = _network("kMed25A", "kMed25B")
    rng = np.random.default_rng(7)
    wins = [rng.random((4000, 25)).astype(np.float32),
            rng.integers(0, 4, (4000, 25)).astype(np.float32),        # heavy ties
            np.full((10, 25), 3.5, np.float32),
            rng.integers(0, 2, (20000, 25)).astype(np.float32)]       # 0-1 principle sample
    for w in wins:
        v = np.concatenate([w, np.full((len(w), 7), np.inf, np.float32)], axis=1)
        got = _run(net, v)[:, 12]
        want = np.sort(w, axis=1)[:, 12]
        assert np.array_equal(got, want)


def test_full_network_sorts():
    net = _network("kMedianA", "kMedianB")
    rng = np.random.default_rng(3)
    for valid in (1, 7, 13, 25):
        w = rng.random((2000, 32)).astype(np.float32)
        w[:, valid:] = np.inf
        assert np.array_equal(_run(net, w)[:, :valid], np.sort(w[:, :valid], axis=1))
