"""Data-parallel host logic on CPU (gloo, world_size 2).

paper_2312_17241_b200.dist.DataParallel drives a replica object through
sample -> compute_grads -> pack -> ONE all_reduce -> unpack -> update.  Here
the replica computes with the CPU oracle (test infrastructure) laid out in
the same flat exchange buffer as the device model, so the test exercises the
real DataParallel code: batch slicing, loss scaling 2/(G*B*out), the single
all-reduce, the touched-row union and the loss slot.  Checks: both replicas
end bit-identical, and equal to a single-process step on the concatenated
batch within 1e-5.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2312_17241_b200.dist import DataParallel, shard_range

HYP = dict(n_f=64, n_c=256, n_p=4, n_levels=4, n_min=4, n_max=32, n_neurons=16)
B_LOCAL = 96
STEPS = 3


class OracleReplica:
    """TrainState protocol on the CPU oracle, exchange buffer laid out like
    grid_model.Model.grads: [gfeats | gmlp | gconf | touched | loss]."""

    def __init__(self, img, batch, seed=0):
        self.m = O.init_model(O.Hyper(**HYP), seed=seed)
        self.img = img
        self.flat = img.reshape(-1, 3)
        self.h, self.w = img.shape[:2]
        self.B = batch
        self.rng = O.seeded_rng(seed, O.SEED_BATCH)
        self.rank, self.world, self.t = 0, 1, 0
        self.probed = [L for L in self.m.levels if L.conf is not None]
        self.n_feat = sum(L.fgrad.size for L in self.m.levels)
        self.n_mlp = sum(w.size + b.size for w, b in zip(self.m.W, self.m.b))
        self.n_conf = sum(L.cgrad.size for L in self.probed)
        self.n_rows = sum(L.conf.shape[0] for L in self.probed)
        self.buf = torch.zeros(self.n_feat + self.n_mlp + self.n_conf + self.n_rows + 1)
        self.loss_sum = torch.zeros(1, dtype=torch.float64)
        z = np.zeros_like
        self.opt = {id(a): (z(a), z(a)) for a in self.m.W + self.m.b + [L.feats for L in self.m.levels]}
        self.copt = {id(L): (z(L.conf), z(L.conf)) for L in self.probed}
        self.touched = [np.zeros(L.conf.shape[0], bool) for L in self.probed]

    def shard(self, rank, world):
        self.rank, self.world = rank, world

    def sample_batch(self):
        pix = O.sample_pixels(self.rng, self.B * self.world, self.w, self.h)
        pix = pix[self.rank * self.B:(self.rank + 1) * self.B]
        return O.pixel_coords(pix, self.w, self.h, np.float32), self.flat[pix]

    def compute_grads(self, xs, targets):
        m = self.m
        y, tr = O.encode_forward(m, xs)
        out, cache = O.mlp_forward(m.W, m.b, y)
        diff = out - targets
        self.loss_sum += float(np.sum(diff.astype(np.float64) ** 2))
        dpred = diff * np.float32(2.0 / (self.world * self.B * 3))
        dy = O.mlp_backward(m.W, m.Wg, m.bg, cache, dpred)
        O.encode_backward(m, tr, dy)
        k = 0
        for L, trl in zip(m.levels, tr):
            if L.conf is not None:
                self.touched[k][np.unique(trl.row)] = True
                k += 1

    def _views(self):
        parts = [L.fgrad for L in self.m.levels] + [a for w, b in zip(self.m.Wg, self.m.bg) for a in (w, b)]
        parts += [L.cgrad for L in self.probed]
        return parts

    def exchange_buffer(self):
        return self.buf

    def pack_exchange(self):
        vals = [torch.from_numpy(p.ravel().astype(np.float32)) for p in self._views()]
        vals += [torch.from_numpy(t.astype(np.float32)) for t in self.touched]
        vals.append(self.loss_sum.float())
        self.buf.copy_(torch.cat(vals))

    def unpack_exchange(self):
        off = 0
        for p in self._views():
            p.ravel()[:] = self.buf[off:off + p.size].numpy()
            off += p.size
        for t in self.touched:
            t[:] = self.buf[off:off + t.size].numpy() > 0
            off += t.size
        self.loss_sum.copy_(self.buf[off:off + 1].double())

    def apply_updates(self):
        m = self.m
        for p, g in zip(m.W + m.b + [L.feats for L in m.levels],
                        m.Wg + m.bg + [L.fgrad for L in m.levels]):
            mm, vv = self.opt[id(p)]
            O.adam_update(p, g, mm, vv, self.t, 1e-2)
            g[:] = 0
        for L, t in zip(self.probed, self.touched):
            rows = np.nonzero(t)[0].astype(np.int32)
            mm, vv = self.copt[id(L)]
            O.CBackend.adam_rebake_rows(L.conf, mm, vv, L.baked, rows, L.cgrad[rows], self.t,
                                        1e-2, 0.9, 0.99, 1e-15)
            L.cgrad[:] = 0
            t[:] = False

    def loss_value(self):
        return float(self.loss_sum[0]) / (self.world * self.B * 3)

    def finish_step(self):
        loss = self.loss_value()
        if not np.isfinite(loss):
            self.t -= 1
            raise FloatingPointError(f"non-finite loss at step {self.t}")
        return loss

    def state(self):
        m = self.m
        return [L.feats.copy() for L in m.levels] + [L.conf.copy() for L in self.probed] + \
               [L.baked.copy() for L in self.probed] + [w.copy() for w in m.W + m.b]


def _image():
    return np.random.default_rng(5).random((20, 20, 3)).astype(np.float32)


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rep = OracleReplica(_image(), B_LOCAL)
    dp = DataParallel(rep, dist)
    losses = [dp.step() for _ in range(STEPS)]
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), losses=np.array(losses),
             **{f"s{i}": a for i, a in enumerate(rep.state())})
    dist.destroy_process_group()


class _SoloDist:
    class ReduceOp:
        SUM = None

    @staticmethod
    def get_rank(group=None):
        return 0

    @staticmethod
    def get_world_size(group=None):
        return 1

    @staticmethod
    def all_reduce(t, op=None, group=None):
        return t


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_replicas_match_single_process_global_batch(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    # replicas are bit-identical (one all-reduce, identical updates)
    for k in r0.files:
        np.testing.assert_array_equal(r0[k], r1[k])
    # ... and equal one process stepping the concatenated global batch
    solo = OracleReplica(_image(), B_LOCAL * world)
    dp = DataParallel(solo, _SoloDist)
    losses = [dp.step() for _ in range(STEPS)]
    np.testing.assert_allclose(r0["losses"], losses, rtol=1e-6)
    for i, a in enumerate(solo.state()):
        if a.dtype == np.uint8:
            assert (r0[f"s{i}"] != a).mean() <= 0.01
        else:
            np.testing.assert_allclose(r0[f"s{i}"], a, rtol=1e-5, atol=2e-2 if i >= 4 else 1e-6)


def test_solo_dataparallel_equals_plain_oracle_step():
    """world=1 DataParallel is exactly the reference step (trainer.py:118-171)."""
    img = _image()
    rep = OracleReplica(img, 128)
    dp = DataParallel(rep, _SoloDist)
    ref = O.TrainState(O.init_model(O.Hyper(**HYP), 0), img, O.TrainCfg(batch_size=128, seed=0))
    for _ in range(STEPS):
        # the loss rides the exchange buffer as one fp32 slot
        assert dp.step() == pytest.approx(ref.step(), rel=1e-7)
    for L, R in zip(rep.m.levels, ref.model.levels):
        np.testing.assert_array_equal(L.feats, R.feats)


@pytest.mark.parametrize("n,world", [(10, 3), (1 << 20, 8), (7, 8), (0, 2)])
def test_shard_range_covers_queries_once(n, world):
    got = []
    for r in range(world):
        lo, hi = shard_range(n, r, world)
        got.extend(range(lo, hi))
    assert got == list(range(n))
