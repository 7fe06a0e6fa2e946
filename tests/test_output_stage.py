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


PNG_TOOL = os.path.join(ROOT, "oracle", "_ref", "png_tool")


@pytest.mark.parametrize("shape,kind", [((7, 5), "noise"), ((1, 1), "noise"), ((64, 96), "ramp"),
                                        ((33, 17), "flat"), ((120, 200), "noise")])
def test_write_png_bytes_match_reference(b200_host, tmp_path, shape, kind):
    """write_png (map_io.cpp:203-260): signature, IHDR, zlib-6 IDAT, IEND and
    CRCs byte for byte against the reference's writer."""
    if not os.path.exists(PNG_TOOL):
        pytest.skip("oracle png_tool not built")
    h, w = shape
    rng = np.random.default_rng(h * 31 + w)
    if kind == "noise":
        rgb = rng.integers(0, 256, (h, w, 3), dtype=np.uint8)
    elif kind == "ramp":
        rgb = np.stack(np.broadcast_arrays((np.arange(w)[None, :] * 255 // max(w - 1, 1)),
                                           (np.arange(h)[:, None] * 255 // max(h - 1, 1)),
                                           np.full((h, w), 77)), -1).astype(np.uint8)
    else:
        rgb = np.full((h, w, 3), 200, np.uint8)
    a, b = tmp_path / "b200.png", tmp_path / "ref.png"
    b200_host.write_png(str(a), rgb)
    subprocess.run([PNG_TOOL, str(b), str(w), str(h)], input=rgb.tobytes(), check=True)
    assert a.read_bytes() == b.read_bytes()
    assert a.read_bytes()[:8] == b"\x89PNG\r\n\x1a\n"


def test_write_png_decodes(b200_host, tmp_path):
    """The stream is a valid PNG: inflate the IDAT and recover the pixels."""
    import struct
    import zlib
    rgb = np.random.default_rng(3).integers(0, 256, (9, 13, 3), dtype=np.uint8)
    p = tmp_path / "x.png"
    b200_host.write_png(str(p), rgb)
    data = p.read_bytes()[8:]
    chunks = {}
    while data:
        n, = struct.unpack(">I", data[:4])
        typ, body, crc = data[4:8], data[8:8 + n], data[8 + n:12 + n]
        assert struct.unpack(">I", crc)[0] == zlib.crc32(typ + body)
        chunks[typ] = body
        data = data[12 + n:]
    assert struct.unpack(">IIBB", chunks[b"IHDR"][:10]) == (13, 9, 8, 2)
    raw = np.frombuffer(zlib.decompress(chunks[b"IDAT"]), np.uint8).reshape(9, 1 + 13 * 3)
    assert (raw[:, 0] == 0).all()
    assert np.array_equal(raw[:, 1:].reshape(9, 13, 3), rgb)
    assert chunks[b"IEND"] == b""


def test_write_png_error(b200_host):
    from paper_2112_00821_b200 import InvalidInputError
    with pytest.raises(InvalidInputError):
        b200_host.write_png("/nonexistent-dir/x.png", np.zeros((2, 2, 3), np.uint8))


@pytest.mark.gpu
def test_viz_png_pipeline_matches_reference(b200, oracle, tmp_path):
    """The CLI's --viz output (tools/fassmvs.cpp:187-196): device colorize of
    the three maps, then write_png, byte-identical to colorize + write_png of
    the reference."""
    if not os.path.exists(PNG_TOOL):
        pytest.skip("oracle png_tool not built")
    rng = np.random.default_rng(11)
    h, w = 48, 64
    d = rng.uniform(4.0, 40.0, (h, w)).astype(np.float32)
    d[rng.random((h, w)) < 0.1] = 0.0
    n = rng.normal(size=(h, w, 3)).astype(np.float32)
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    c = rng.uniform(0, 1, (h, w)).astype(np.float32)
    for name, got, want in [("depth", b200.colorize_depth(d, 4.0, 40.0), oracle.colorize_depth(d, 4.0, 40.0)),
                            ("normal", b200.colorize_normals(n), oracle.colorize_normals(n)),
                            ("conf", b200.colorize_confidence(c), oracle.colorize_confidence(c))]:
        a, b = tmp_path / f"{name}_b200.png", tmp_path / f"{name}_ref.png"
        b200.write_png(str(a), got)
        subprocess.run([PNG_TOOL, str(b), str(w), str(h)], input=np.ascontiguousarray(want).tobytes(),
                       check=True)
        assert a.read_bytes() == b.read_bytes(), name
