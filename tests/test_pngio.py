"""PNG output (pngio.py:34-41 contract) on the host: the numpy quantisation
rule, the writer read back by Pillow (the reference's reader) and by our own
reader, Pillow-written files (adaptive filters) read back, error types."""
import numpy as np
import pytest

from paper_2312_17241_b200 import UnsupportedFormat
from paper_2312_17241_b200.pngio import encode_png, load_image, quantize, save_image


def test_quantize_matches_reference_rule():
    px = np.random.default_rng(0).uniform(-0.2, 1.2, (17, 23, 3)).astype(np.float32)
    px[0, 0] = [0.5 / 255, 1.5 / 255, 254.5 / 255]            # round-half-even cases
    np.testing.assert_array_equal(quantize(px), np.rint(np.clip(px, 0.0, 1.0) * 255.0).astype(np.uint8))


def test_png_round_trip_and_pillow(tmp_path):
    PIL = pytest.importorskip("PIL.Image")
    px = np.random.default_rng(1).random((31, 47, 3)).astype(np.float32)
    path = str(tmp_path / "a.png")
    save_image(path, px)
    want = quantize(px)
    with PIL.open(path) as im:
        np.testing.assert_array_equal(np.asarray(im.convert("RGB")), want)
    np.testing.assert_array_equal(load_image(path), want.astype(np.float32) / 255.0)
    # Pillow's own encoder (adaptive filters), RGBA and grayscale files
    for mode, arr in (("RGB", want), ("RGBA", np.dstack([want, np.full(want.shape[:2], 7, np.uint8)])),
                      ("L", want[:, :, 0])):
        p2 = str(tmp_path / f"pil_{mode}.png")
        PIL.fromarray(arr, mode=mode).save(p2, format="PNG")
        rgb = want if mode != "L" else np.repeat(want[:, :, :1], 3, axis=2)
        np.testing.assert_array_equal(load_image(p2), rgb.astype(np.float32) / 255.0)
    assert encode_png(want)[:8] == b"\x89PNG\r\n\x1a\n"


def test_png_errors(tmp_path):
    with pytest.raises(UnsupportedFormat):
        save_image(str(tmp_path / "x.png"), np.zeros((4, 4), np.float32))
    bad = tmp_path / "bad.png"
    bad.write_bytes(b"not a png")
    with pytest.raises(UnsupportedFormat):
        load_image(str(bad))
