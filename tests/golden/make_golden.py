"""Generates the golden fixtures of tests/golden/ from the parity oracle
(the unmodified reference built against the Eigen shim, oracle/_ref).

    python tests/golden/make_golden.py

Each fixture is a small end-to-end estimate_bundle case: the inputs are
regenerated deterministically by the oracle's own render_scene (seed 1), the
stored outputs are the oracle's depth / normals / confidence. The GPU tests
compare the B200 library against these files when the oracle library is not
available on the box; tests/test_oracle.py checks the oracle still
reproduces them.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_2112_00821_b200 import (CostFunctionSpec, CostKind, PipelineConfig, SgmConfig,  # noqa: E402
                                   SgmVariant)

CASES = {
    # smoke(): slanted 128x96, 2 levels, census 5x5, Pi-sn (as __graft_entry__.smoke)
    "smoke": (dict(kind="slanted", w=128, h=96, focal=128.0, depth=10.0, views=5, step=0.5,
                   tilt=30.0, texture=0.2),
              dict(d_min=4.0, d_max=40.0, levels=2, max_planes=128, cost="census5", variant="sn")),
    # acceptance criterion 4 scene at half size (acceptance.cpp:265-304)
    "c4_fronto_ncc": (dict(kind="fronto", w=160, h=120, focal=160.0, depth=10.0, views=5, step=0.5,
                           tilt=0.0, texture=0.35),
                      dict(d_min=8.0, d_max=14.0, levels=1, max_planes=256, cost="ncc5",
                           variant="plane")),
    # C2 shape at 1/10 scale
    "census_sn_3lvl": (dict(kind="slanted", w=192, h=108, focal=192.0, depth=10.0, views=5,
                            step=0.59, tilt=30.0, texture=0.2),
                       dict(d_min=4.0, d_max=40.0, levels=3, max_planes=128, cost="census5",
                            variant="sn")),
}


def case(backend, name):
    scene, c = CASES[name]
    bundle, _, _ = backend.render_plane_scene(scene["kind"], scene["w"], scene["h"], scene["focal"],
                                              scene["depth"], scene["views"], scene["step"], seed=1,
                                              tilt_deg=scene["tilt"], texture_scale=scene["texture"])
    kinds = {"census5": (CostKind.CensusHamming, 5, 5), "ncc5": (CostKind.NccTruncated, 5, 5)}
    variants = {"plane": SgmVariant.Plane, "sn": SgmVariant.SurfaceNormal,
                "pg": SgmVariant.PathGradient}
    cfg = PipelineConfig(c["d_min"], c["d_max"], pyramid_levels=c["levels"],
                         max_planes=c["max_planes"], sgm=SgmConfig(variant=variants[c["variant"]]),
                         cost=CostFunctionSpec(*kinds[c["cost"]]))
    return bundle, cfg


def main():
    import ref
    oracle = ref.load()
    for name in CASES:
        bundle, cfg = case(oracle, name)
        r = oracle.estimate_bundle(bundle, cfg)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), depth=r.depth, normals=r.normals,
                            confidence=r.confidence)
        print(name, r.depth.shape, float((r.depth > 0).mean()))


if __name__ == "__main__":
    main()
