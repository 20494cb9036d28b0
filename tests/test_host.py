"""CPU-only checks of the host side: the C-ABI library loads and exports every
symbol include/probegrid_b200.h declares, and the host mirror of the
reference interface (hyper-parameters, level ladder, initial values) agrees
with the oracle exactly.  No kernel is called (no GPU here)."""

import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2312_17241_b200 import _lib
from paper_2312_17241_b200.errors import InvalidHyperparameter
from paper_2312_17241_b200.hyper import (HyperParams, LevelMode, build_level_specs, grid_struct,
                                         level_resolution, mlp_struct)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "probegrid_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const char \*|int64_t |int )(pg_\w+)\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 30
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(declared) == sorted(_lib.exported_symbols())
    assert b"sm_100a" in lib.pg_version()


def test_struct_layouts_match_header():
    import ctypes
    assert ctypes.sizeof(_lib.PgGrid) == 4 * (6 + 3 * 64 + 6)
    assert ctypes.sizeof(_lib.PgMlp) == 4 * (1 + 18)


@pytest.mark.parametrize("kw", [dict(), dict(n_f=2**12, n_c=2**14, n_p=4),
                                dict(n_f=2**16, n_c=2**16, n_p=8, n_max=8192),
                                dict(n_f=2**8, n_c=2**16, n_p=4, d=3),
                                dict(n_levels=3, n_min=4, n_max=16, n_f=32)])
def test_level_ladder_matches_oracle(kw):
    h = HyperParams(**kw)
    specs = build_level_specs(h.n_min, h.n_max, h.n_levels, h.n_f, h.d)
    oh = O.Hyper(**kw)
    assert [(s.resolution, s.mode is LevelMode.DENSE) for s in specs] == O.level_ladder(oh)


def test_level_resolution_kats():
    # test_indexing.py:36-42
    assert level_resolution(3, 16, 512, 16) == 32
    assert level_resolution(0, 16, 512, 16) == 16
    assert level_resolution(15, 16, 512, 16) == 512


@pytest.mark.parametrize("bad", [dict(n_f=100), dict(n_p=3), dict(n_p=512, n_f=1024),
                                 dict(n_f=4, n_p=8), dict(d=4), dict(n_levels=0),
                                 dict(n_min=0), dict(out_dim=0), dict(feature_dim=17)])
def test_invalid_hyperparameters(bad):
    with pytest.raises(InvalidHyperparameter):
        HyperParams(**bad).validate()


def test_grid_struct_kinds_and_slots():
    h = HyperParams(n_f=2**12, n_c=2**14, n_p=4)
    specs = build_level_specs(h.n_min, h.n_max, h.n_levels, h.n_f, h.d)
    probed = [s.level for s in specs if s.mode is LevelMode.HASHED]
    g = grid_struct(h, specs, probed)
    assert [g.kind[i] for i in range(16)] == [0] * 6 + [2] * 10
    assert [g.slot[i] for i in range(16)] == [-1] * 6 + list(range(10))
    assert g.log2_np == 2 and g.n_f == 4096 and g.n_c == 16384
    assert list(g.primary) == [1, 2654435761, 805459861]
    m = mlp_struct(h.mlp_widths())
    assert m.n_layers == 3 and list(m.widths[:4]) == [32, 64, 64, 3]


@pytest.mark.parametrize("kw,seed,dtype", [(dict(n_f=32, n_c=64, n_p=4, n_levels=3, n_min=4,
                                                 n_max=16, n_neurons=8), 0, np.float32),
                                           (dict(n_f=2**12, n_c=2**14, n_p=4), 3, np.float32),
                                           (dict(n_f=16, n_c=8, n_p=4, n_levels=2, n_min=4,
                                                 n_max=8), 1, np.float64)])
def test_host_initial_values_match_oracle(kw, seed, dtype):
    from paper_2312_17241_b200.grid_model import host_init_arrays
    h = HyperParams(**kw)
    specs = build_level_specs(h.n_min, h.n_max, h.n_levels, h.n_f, h.d)
    probed = {s.level for s in specs if s.mode is LevelMode.HASHED and h.n_p > 1}
    feats, conf, W, B = host_init_arrays(h, seed, dtype, probed)
    om = O.init_model(O.Hyper(**kw), seed=seed, dtype=dtype)
    for L in om.levels:
        np.testing.assert_array_equal(feats[L.level], L.feats)
        if L.conf is not None:
            np.testing.assert_array_equal(conf[L.level], L.conf)
        else:
            assert L.level not in conf
    for a, b in zip(W, om.W):
        np.testing.assert_array_equal(a, b)


def test_product_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2312_17241_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in text.replace("oracle (", ""), f


def test_round2_host_rules():
    """Host-side rules of the round-2 paths: feature-gradient replicas by
    probing ranges per level, the cell-cache budgets, the bench's operation
    and byte counts."""
    import os
    import bench
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200 import train
    f32 = np.float32
    assert train.grad_replicas(pg.HyperParams(n_f=2**12, n_c=2**14, n_p=4), f32) == 1      # 1024 ranges
    assert train.grad_replicas(pg.HyperParams(n_f=2**8, n_c=2**12, n_p=16), f32) == 8      # 16 ranges
    assert train.grad_replicas(pg.HyperParams(), f32) == 1                                 # 4 ranges: warp-aggregated
    assert train.grad_replicas(pg.HyperParams(n_f=2**8, n_c=2**12, n_p=4), np.float64) == 1
    os.environ["PG_TRAIN_REPS"] = "3"
    try:
        assert train.grad_replicas(pg.HyperParams(), f32) == 3
    finally:
        del os.environ["PG_TRAIN_REPS"]
    assert train.train_cell_budget() == 32 << 20
    h = pg.HyperParams(**bench.C1)
    assert bench.train_l2_ops_per_sample(h, 10) == 328
    assert bench.train_bytes_per_sample(h, 10) == 6840          # C1 6,840 B/sample
    assert bench.infer_bytes_per_query(pg.HyperParams(**bench.C2), 9, 4) == 312
    from paper_2312_17241_b200 import decode
    if "PG_DECODE_CELL_MB" not in os.environ:
        assert decode.CELL_BUDGET == 96 << 20


def test_training_tile_swizzle_is_bank_conflict_free():
    """Restates pg_train_mma.cu's tile layout (row stride kS = 72 floats,
    column ^ 12 in rows with bit 2 set: sw()) and checks the three warp access
    patterns it is designed for hit 32 distinct banks: fragment walks over 4
    rows x 8 columns (P1) and 8 rows x 4 columns (P2, the weight-gradient and
    W^T GEMMs), and the C-fragment stores (rows 2c / 2c+1, columns g)."""
    kS = 72

    def sw(r, c):
        return r * kS + (c ^ ((r & 4) * 3))

    def distinct(cells):
        banks = [sw(r, c) % 32 for r, c in cells]
        return len(set(banks)) == 32

    for R in range(0, 64, 4):
        for C in range(0, 64, 8):
            assert distinct([(R + c, C + g) for c in range(4) for g in range(8)])
    for R in range(0, 64, 8):
        for C in range(0, 64, 4):
            assert distinct([(R + g, C + c) for g in range(8) for c in range(4)])
        for C in range(0, 64, 8):
            for e in (0, 1):
                assert distinct([(R + 2 * c + e, C + g) for c in range(4) for g in range(8)])
    # the swizzle permutes columns within each row (a bijection on [0, 64))
    for r in range(64):
        assert sorted(sw(r, c) - r * kS for c in range(64)) == list(range(64))


def test_decode_output_index_reciprocal():
    """pg_decode_tc.cu splits the output index i into (query, column) with
    q = (i * ceil(2^16 / od)) >> 16: exact for every i < 128 * od it sees."""
    for od in range(1, 5):
        mag = (65536 + od - 1) // od
        for i in range(128 * od):
            assert (i * mag) >> 16 == i // od
