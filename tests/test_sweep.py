"""Sweep harness, metrics and size-budgeted hyper-parameters on the host
(sweep.py, metrics.py, trainer.py:245-281 of the reference; SURVEY 8(f)
row 3).  select_hyperparams is pinned against the REAL reference's choices
(tests/golden/cngp_files.npz); the rank dealing of run_sweep is exercised
with gloo, world 2, and a stand-in fit (the GPU fits are in test_gpu_sweep)."""

import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2312_17241_b200 as pg
from paper_2312_17241_b200 import sweep
from paper_2312_17241_b200.model_io import size_report

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "cngp_files.npz"))


def test_select_hyperparams_matches_reference():
    for t, n_f, n_c, n_p, total in GOLD["select_hyperparams"]:
        h = pg.select_hyperparams(int(t))
        assert (h.n_f, h.n_c, h.n_p) == (n_f, n_c, n_p)
        assert size_report(h).total_bytes == total <= max(t, total)


def test_select_hyperparams_limits():
    floor = size_report(pg.HyperParams(n_f=2**6, n_c=2**10, n_p=2)).total_bytes
    assert (pg.select_hyperparams(floor).n_f, pg.select_hyperparams(floor).n_c) == (2**6, 2**10)
    with pytest.raises(pg.TargetTooSmall):
        pg.select_hyperparams(1000)
    for target in [25_000, 60_000, 300_000, 5_000_000]:
        assert size_report(pg.select_hyperparams(target)).total_bytes <= target
    rep = size_report(pg.select_hyperparams(150_000))
    assert abs(math.log2(rep.feature_bytes / (rep.total_bytes / 3))) <= 1.0
    assert abs(math.log2(rep.index_bytes / (2 * rep.total_bytes / 3))) <= 1.0


def test_psnr_and_pareto_front():
    a = np.random.default_rng(0).random((8, 8, 3))
    assert pg.psnr(a, a) == float("inf")
    assert abs(pg.psnr(a, a + 0.1) - 20.0) < 1e-9
    with pytest.raises(pg.DimensionMismatch):
        pg.psnr(a, a[:4])
    pts = [(100, 30.0), (100, 31.0), (200, 30.5), (200, 35.0), (300, 35.0), (50, 20.0), (300, 36.0)]
    assert pg.pareto_front(pts) == [(50, 20.0), (100, 31.0), (200, 35.0), (300, 36.0)]
    assert pg.pareto_front([(1, 2.0), (1, 2.0)]) == [(1, 2.0), (1, 2.0)]   # ties kept


def test_expand_grid_and_csv(tmp_path):
    base = pg.HyperParams(n_levels=4, n_min=4, n_max=16, n_neurons=16)
    grid = pg.expand_grid(base, [64, 128], [256], [1, 4], levels=[4, 6])
    assert len(grid) == 8 and {(h.n_f, h.n_p, h.n_levels) for h in grid} == \
        {(f, p, lv) for f in (64, 128) for p in (1, 4) for lv in (4, 6)}
    with pytest.raises(pg.InvalidHyperparameter):
        pg.expand_grid(base, [], [256], [4])
    with pytest.raises(pg.InvalidHyperparameter):
        pg.expand_grid(base, [64], [256], [3])           # n_p not a power of two
    pts = [sweep.SweepPoint("probed", 64, 256, 4, 4, 16, 0, 1234, float("inf"), 1.5),
           sweep.SweepPoint("baseline", 64, 256, 1, 4, 16, 1, 999, 31.25, 0.25)]
    path = str(tmp_path / "s.csv")
    pg.write_csv(pts, path)
    lines = open(path).read().splitlines()
    assert lines[0] == ",".join(sweep.CSV_COLUMNS)
    assert lines[1] == "probed,64,256,4,4,16,0,1234,inf,1.500"
    assert lines[2] == "baseline,64,256,1,4,16,1,999,31.2500,0.250"


class _FakeResult:
    def __init__(self, hyper, seed):
        self.final_psnr = float(seed) + hyper.n_p
        self.ms_per_step = 1.0
        self.size_report = size_report(hyper)


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2312_17241_b200.train as tr
    ran = []
    tr.fit = lambda img, h, cfg: (ran.append((h.n_p, cfg.seed)), _FakeResult(h, cfg.seed))[1]
    base = pg.HyperParams(n_levels=4, n_min=4, n_max=16, n_neurons=16)
    grid = pg.expand_grid(base, [64], [256], [1, 2, 4])
    pts = pg.run_sweep(None, grid, [0, 1], pg.TrainConfig(steps=1), dist=dist)
    np.save(os.path.join(out, f"r{rank}.npy"),
            np.array([[p.n_p, p.seed, p.psnr_db, p.method == "baseline"] for p in pts] + [[-1, -1, -1, -1]] +
                     [[n, s, 0, 0] for n, s in ran]))
    dist.destroy_process_group()


def test_run_sweep_deals_jobs_to_ranks(tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (np.load(str(tmp_path / f"r{i}.npy")) for i in (0, 1))
    sep0, sep1 = int(np.where(r0[:, 0] == -1)[0][0]), int(np.where(r1[:, 0] == -1)[0][0])
    np.testing.assert_array_equal(r0[:sep0], r1[:sep1])              # every rank returns the full list
    want = [(p, sd) for p in (1, 2, 4) for sd in (0, 1)]              # product order
    assert [tuple(map(int, x[:2])) for x in r0[:sep0]] == want
    assert [bool(x[3]) for x in r0[:sep0]] == [p == 1 for p, _ in want]
    ran0 = {tuple(map(int, x[:2])) for x in r0[sep0 + 1:]}
    ran1 = {tuple(map(int, x[:2])) for x in r1[sep1 + 1:]}
    assert ran0 | ran1 == set(want) and not ran0 & ran1               # each job ran exactly once
