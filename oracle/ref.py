"""Python binding of the parity oracle (TEST INFRASTRUCTURE ONLY).

The oracle is the UNMODIFIED reference library (/root/reference/proj/src)
compiled in place against oracle/eigen_shim by oracle/Makefile into
oracle/_ref/libfassmvs_ref.so, with the C ABI of include/fmvs.h exported under
the ``ref_`` prefix by oracle/ref_capi.cpp. It is bound with the product's
own Python API class so a test reads ``oracle.sweep_cost_volume(...)`` and
``b200.sweep_cost_volume(...)`` identically.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libfassmvs_ref.so")
REFERENCE = "/root/reference/proj"


def build(quiet: bool = True) -> bool:
    """Builds oracle/_ref when the reference sources are present."""
    if not os.path.isdir(REFERENCE):
        return os.path.exists(LIB)
    cmd = ["make", "-C", HERE, "-j8", "all", "tests"]
    r = subprocess.run(cmd, capture_output=quiet, text=True)
    if r.returncode != 0:
        raise RuntimeError("oracle build failed:\n" + (r.stdout or "") + (r.stderr or ""))
    return True


def available() -> bool:
    return os.path.exists(LIB)


def load():
    """The oracle as a paper_2112_00821_b200.fassmvs.Backend (prefix ref_)."""
    from paper_2112_00821_b200 import _abi
    from paper_2112_00821_b200.fassmvs import Backend
    if not available():
        raise FileNotFoundError(f"oracle library missing: {LIB} (make -C oracle)")
    return Backend(LIB, "ref_", extras=_abi.ORACLE_EXTRAS, needs_context=False)
