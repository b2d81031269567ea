"""PGM / PNG I/O (image.py:69-129) against files the reference wrote and read (CPU)."""

import numpy as np
import pytest

from paper_1603_08109_b200 import (ParameterError, load_image, load_pgm, quantize, read_raster, save_image,
                                   save_pgm, write_raster)


def test_save_pgm_bytes_equal_reference(tools_golden, tmp_path):
    for tag in ("edge", "rand"):
        p = tmp_path / f"{tag}.pgm"
        save_pgm(p, tools_golden[f"io_{tag}_in"])
        assert np.array_equal(np.frombuffer(p.read_bytes(), np.uint8), tools_golden[f"io_{tag}_pgm"]), tag


def test_quantize_matches_reference_rounding(tools_golden):
    # the edge row holds -3, 0.49, 0.5, 254.5, 300, 127.5, 1.4999999999, 2.5000000001, 255, 0
    pgm = tools_golden["io_edge_pgm"]
    q = quantize(tools_golden["io_edge_in"])
    assert q.dtype == np.uint8 and np.array_equal(q.ravel(), pgm[-q.size:])


@pytest.mark.parametrize("name", ["comment", "multi_comment", "crlf_ws"])
def test_load_pgm_headers(name, tools_golden, tmp_path):
    p = tmp_path / f"{name}.pgm"
    p.write_bytes(tools_golden[f"io_hdr_{name}"].tobytes())
    ref = tools_golden[f"io_hdr_{name}_loaded"]
    out = load_pgm(p)
    assert out.dtype == np.float64 and np.array_equal(out, ref)
    raster = read_raster(p)
    assert raster.dtype == np.uint8 and np.array_equal(raster, ref)


@pytest.mark.parametrize("name", ["wrong_magic", "maxval", "no_dims", "garbage"])
def test_load_pgm_errors(name, tools_golden, tools_scalars, tmp_path):
    p = tmp_path / f"{name}.pgm"
    p.write_bytes(tools_golden[f"io_bad_{name}"].tobytes())
    with pytest.raises(ValueError) as ei:
        load_pgm(p)
    assert str(ei.value) == tools_scalars["io_errors"][name].replace("{path}", str(p))


def test_truncated_raster(tmp_path):
    p = tmp_path / "t.pgm"
    p.write_bytes(b"P5\n4 4\n255\n\x00\x01")
    with pytest.raises(ValueError):
        load_pgm(p)


def test_png_written_by_reference(tools_golden, tmp_path):
    p = tmp_path / "r.png"
    p.write_bytes(tools_golden["io_png_bytes"].tobytes())
    assert np.array_equal(load_image(p), tools_golden["io_png_loaded"])
    assert np.array_equal(read_raster(p), tools_golden["io_png_loaded"])


def test_roundtrips(tmp_path, random_image):
    img = random_image(7, 11)
    for name in ("a.pgm", "a.png"):
        save_image(tmp_path / name, img)
        assert np.array_equal(load_image(tmp_path / name), img)
    write_raster(tmp_path / "b.pgm", img.astype(np.uint8))
    assert np.array_equal(load_pgm(tmp_path / "b.pgm"), img)


def test_save_rejects_non_finite(tmp_path):
    with pytest.raises(ParameterError):
        save_pgm(tmp_path / "x.pgm", np.array([[1.0, np.nan]]))
