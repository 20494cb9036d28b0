"""The .cngp format layer on the host (model_io.py:40-277, FORMAT.md):
header / size accounting / index packing / typed errors, pinned against
files written by the REAL reference (tests/golden/cngp_files.npz, made by
tests/golden/make_golden_cngp.py) — mirrors test_model_io.py's
TestBitPacking, TestSizeReport and TestDeserializeErrors."""

import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2312_17241_b200 import model_io as mio
from paper_2312_17241_b200.errors import (BadMagic, InvariantViolation, ModelFileError,
                                          TruncatedFile, VersionMismatch)
from paper_2312_17241_b200.hyper import HyperParams, LevelMode, build_level_specs

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "cngp_files.npz"))
NAMES = ["np4", "np16", "np8_d3", "np2_sig_f4", "np1"]


def _raw(name):
    return bytes(GOLD[f"{name}_file"])


@pytest.mark.parametrize("name", NAMES)
def test_reference_files_parse(name):
    raw = _raw(name)
    kw = {k: v for k, v in GOLD[f"{name}_kw"]}
    pf = mio.parse(raw)
    h = pf.hyper
    for k, v in kw.items():
        assert str(getattr(h, k)) == v, k
    assert mio.size_report(h).total_bytes == len(raw)
    specs = build_level_specs(h.n_min, h.n_max, h.n_levels, h.n_f, h.d)
    want = [s.level for s in specs if s.mode is LevelMode.HASHED] if h.n_p > 1 else []
    assert pf.probed == want
    baked = [mio.unpack_indices(pf.packed[i].tobytes(), h.n_c, h.n_p) for i in range(len(pf.probed))]
    np.testing.assert_array_equal(np.array(baked).reshape(GOLD[f"{name}_baked"].shape),
                                  GOLD[f"{name}_baked"])
    # host re-pack reproduces the reference's index blocks byte for byte
    for i in range(len(pf.probed)):
        assert mio.pack_indices(baked[i], h.n_p) == pf.packed[i].tobytes()


def test_format_md_worked_example():
    raw = bytes(GOLD["format_example_file"])
    assert len(raw) == 87
    h, w, hh = mio.read_header(raw)
    assert (h.d, h.n_levels, h.feature_dim, h.n_f, h.n_c, h.n_p, w, hh) == (2, 1, 1, 4, 8, 2, 3, 2)
    pf = mio.parse(raw)
    np.testing.assert_array_equal(pf.feats16.ravel().astype(np.float32), [0.5, 1.0, -2.0, 0.25])
    assert pf.packed.tobytes() == bytes([0x4D])
    np.testing.assert_array_equal(pf.mlp16.astype(np.float32),
                                  [0.5, 0.5, -1, -1] + [0.5] * 6 + [-1] * 3)


def test_spec_example_byte():
    assert mio.pack_indices(np.array([1, 0, 1, 1, 0, 0, 1, 0], np.uint8), 2) == bytes([0b01001101])


def test_round_trip_various_widths():
    rng = np.random.default_rng(0)
    for n_p in [2, 4, 8, 16, 32, 64, 128, 256]:
        for n_c in [1, 5, 8, 33, 256]:
            e = rng.integers(0, n_p, size=n_c).astype(np.uint8)
            raw = mio.pack_indices(e, n_p)
            assert len(raw) == (n_c * (n_p.bit_length() - 1) + 7) // 8
            np.testing.assert_array_equal(mio.unpack_indices(raw, n_c, n_p), e)


@settings(max_examples=100, deadline=None)
@given(st.lists(st.integers(0, 15), min_size=1, max_size=64))
def test_round_trip_property(values):
    e = np.array(values, dtype=np.uint8)
    np.testing.assert_array_equal(mio.unpack_indices(mio.pack_indices(e, 16), len(values), 16), e)


def test_size_report_formulas():
    h = HyperParams(n_f=2**6, n_c=2**10, n_p=2, n_levels=16, n_min=16, n_max=512)
    assert mio.size_report(h).feature_bytes == 16 * 64 * 2 * 2
    h = HyperParams(n_f=2**6, n_c=2**16, n_p=2**4, n_levels=16, n_min=16, n_max=512)
    assert mio.size_report(h).index_bytes == 16 * (65536 * 4 // 8)
    h = HyperParams(n_f=2**12, n_c=2**10, n_p=2**2, n_levels=16, n_min=16, n_max=512)
    hashed = sum(1 for s in build_level_specs(16, 512, 16, 2**12, 2) if (s.resolution + 1) ** 2 > 2**12)
    assert 0 < hashed < 16 and mio.size_report(h).index_bytes == hashed * (1024 * 2 // 8)
    assert mio.size_report(HyperParams(n_f=64, n_c=256, n_p=1, n_levels=4, n_min=4, n_max=16)).index_bytes == 0


def test_bad_magic():
    raw = bytearray(_raw("np4"))
    raw[:4] = b"NOPE"
    with pytest.raises(BadMagic):
        mio.parse(bytes(raw))


def test_version_mismatch():
    raw = bytearray(_raw("np4"))
    raw[4] = 99
    with pytest.raises(VersionMismatch):
        mio.parse(bytes(raw))


def test_truncation_everywhere():
    raw = _raw("np2_sig_f4")
    for cut in [0, 3, mio.HEADER_BYTES - 1, mio.HEADER_BYTES, mio.HEADER_BYTES + 17, len(raw) // 2,
                len(raw) - 1]:
        with pytest.raises(TruncatedFile):
            mio.parse(raw[:cut])


def test_trailing_garbage():
    with pytest.raises(InvariantViolation):
        mio.parse(_raw("np2_sig_f4") + b"\x00")


def test_invalid_hyperparameters_in_header():
    raw = bytearray(_raw("np2_sig_f4"))
    raw[20:24] = (3).to_bytes(4, "little")  # n_f = 3, not a power of two
    with pytest.raises(InvariantViolation):
        mio.parse(bytes(raw))


def test_unknown_flag_bits():
    raw = bytearray(_raw("np2_sig_f4"))
    raw[11] = 2
    with pytest.raises(InvariantViolation):
        mio.parse(bytes(raw))


@settings(max_examples=200, deadline=None)
@given(st.binary(min_size=0, max_size=200))
def test_fuzzed_headers_never_crash(blob):
    try:
        mio.parse(blob)
    except ModelFileError:
        pass


@settings(max_examples=100, deadline=None)
@given(st.integers(0, 51), st.binary(min_size=1, max_size=4))
def test_fuzzed_header_mutations_never_crash(offset, patch):
    raw = bytearray(bytes(GOLD["format_example_file"]))
    raw[offset:offset + len(patch)] = patch
    try:
        mio.parse(bytes(raw))
    except ModelFileError:
        pass
