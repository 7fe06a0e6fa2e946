"""The drop-in boundary: the C-ABI library loads without a GPU and exports
every entry point include/fmvs.h declares; the oracle exports the same set
under its prefix."""
import ctypes
import os
import re

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fmvs.h")
LIB = os.path.join(ROOT, "paper_2112_00821_b200", "_lib", "libfmvs.so")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(fmvs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    names = declared()
    assert "fmvs_estimate_bundle" in names
    assert "fmvs_estimate_bundle_device" in names
    assert len(names) >= 30


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_oracle_exports_the_same_entry_points(oracle):
    # host-only / context plumbing has no reference analogue
    skip = {"fmvs_ctx_create", "fmvs_ctx_destroy", "fmvs_ctx_synchronize", "fmvs_ctx_level_stats",
            "fmvs_ctx_last_launch_count", "fmvs_ctx_stream", "fmvs_host_alloc", "fmvs_host_free",
            "fmvs_estimate_bundle_device", "fmvs_ctx_set_timing", "fmvs_ctx_stage_count",
            "fmvs_ctx_stage_name", "fmvs_ctx_stage_time", "fmvs_ctx_stage_reset",
            "fmvs_ctx_sweep_stats", "fmvs_current_device",
            # the multi-GPU sequence engine is checked against ref_estimate_sequence
            "fmvs_estimate_sequence_multi", "fmvs_sequence_plan",
            # the reference writers run as oracle/_ref/{pfm,png}_tool (subprocesses)
            "fmvs_write_pfm", "fmvs_write_png"}
    missing = [n for n in declared() if n not in skip and not hasattr(oracle.lib, "ref_" + n[5:])]
    assert not missing, missing


def test_abi_version(b200_host):
    assert b200_host.fn["abi_version"]() == 1


def test_python_binding_fails_loudly_without_library(tmp_path):
    import pytest
    from paper_2112_00821_b200 import Backend
    with pytest.raises(FileNotFoundError):
        Backend(str(tmp_path / "missing.so"), "fmvs_")
