"""Accuracy scoring on the device against the reference's
evaluation.cpp: integer counts, Acc/Cpl/F and the ROC curve must be
bit-identical; the L1 means are FP64 tree sums and are held to 1e-12
relative (the reference sums sequentially in raster order). Quantised
confidences exercise the ROC tie break (raster order)."""
import numpy as np
import pytest

from paper_2112_00821_b200 import InvalidInputError

from scenes import config, render

pytestmark = pytest.mark.gpu

THETAS = (1.25, 1.1, 1.05, 1.01)


def _maps(rng, h=57, w=83):
    gt = rng.uniform(3.0, 30.0, (h, w)).astype(np.float32)
    est = (gt * rng.uniform(0.9, 1.1, (h, w))).astype(np.float32)
    est[rng.random((h, w)) < 0.1] = 0.0
    gt[rng.random((h, w)) < 0.05] = 0.0
    est[0, :3] = [np.nan, np.inf, -2.0]
    gt[1, :2] = [np.inf, -1.0]
    conf = (np.round(rng.uniform(0, 1, (h, w)) * 8) / 8).astype(np.float32)  # many ties
    conf[2, :2] = [-0.0, 0.0]
    return est, gt, conf


def _check(b200, oracle, est, gt, conf):
    a_l1, a_sc = b200.evaluate(est, gt, THETAS)
    b_l1, b_sc = oracle.evaluate(est, gt, THETAS)
    assert a_l1["valid_both"] == b_l1["valid_both"]
    for k in ("l1_abs", "l1_rel"):
        assert a_l1[k] == pytest.approx(b_l1[k], rel=1e-12), k
    assert a_sc == b_sc  # counts and the ratios derived from them: exact
    for theta in (1.05, 1.25):
        a_d, a_e = b200.roc_curve(est, gt, conf, theta)
        b_d, b_e = oracle.roc_curve(est, gt, conf, theta)
        assert np.array_equal(a_d, b_d) and np.array_equal(a_e, b_e), theta


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_evaluation_random_maps(b200, oracle, seed):
    est, gt, conf = _maps(np.random.default_rng(seed))
    _check(b200, oracle, est, gt, conf)


def test_evaluation_of_a_pipeline_result(b200, oracle):
    bundle, gd, _ = render(oracle, "slanted", 128, 96, tilt=30.0, step=0.5, texture=0.3)
    r = b200.estimate_bundle(bundle, config(4.0, 40.0, levels=2, cost="census5", max_planes=64))
    _check(b200, oracle, r.depth, gd[2], r.confidence)


def test_evaluation_errors(b200, oracle):
    z = np.zeros((4, 5), np.float32)
    o = np.ones((4, 5), np.float32)
    for be in (b200, oracle):
        with pytest.raises(InvalidInputError):
            be.evaluate(z, o)  # no pixel valid in both
        with pytest.raises(InvalidInputError):
            be.roc_curve(z, o, o)  # no valid estimates
        with pytest.raises(InvalidInputError):
            be.evaluate(o, o[:, :4])
