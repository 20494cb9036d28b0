"""Data-parallel training on the GPU path (dist.DataParallel around the
device TrainState): two replicas with the gloo backend sharing cuda:0 — a
functional check of the step the driver runs with NCCL on N GPUs (the
all-reduce is host-staged here; nothing waits on another rank's kernels).
Checks: replicas bit-identical after several steps; one DP step equals a
single-process step on the concatenated global batch within 1e-5."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HYP = dict(n_f=2**12, n_c=2**14, n_p=4)
B_LOCAL = 4096


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _image():
    from tests.golden_util import smooth_image
    return smooth_image(64, 64)


def _snapshot(st):
    m = st.model
    return {"dense": m.dense.cpu().numpy().copy(), "conf": m.conf.cpu().numpy().copy(),
            "baked": m.baked.cpu().numpy().copy(), "loss": st.loss_value()}


def _worker(rank, world, port, out, steps):
    import torch.distributed as dist
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200.dist import DataParallel
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    st = pg.TrainState(pg.init_model(pg.HyperParams(**HYP), seed=0), _image(),
                       pg.TrainConfig(batch_size=B_LOCAL, seed=0), exact_mlp=True)
    dp = DataParallel(st, dist)
    for i in range(steps):
        dp.launch_step()
        if i == 0:
            np.savez(os.path.join(out, f"step1_rank{rank}.npz"), **_snapshot(st))
    torch.cuda.synchronize()
    np.savez(os.path.join(out, f"rank{rank}.npz"), **_snapshot(st))
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def dp_run(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    out = str(tmp_path_factory.mktemp("dp"))
    mp.spawn(_worker, args=(2, _free_port(), out, 4), nprocs=2, join=True)
    return out


def test_replicas_stay_bit_identical(dp_run):
    a = np.load(os.path.join(dp_run, "rank0.npz"))
    b = np.load(os.path.join(dp_run, "rank1.npz"))
    for k in ("dense", "conf", "baked", "loss"):
        np.testing.assert_array_equal(a[k], b[k])


def test_one_dp_step_equals_global_batch_step(dp_run):
    import paper_2312_17241_b200 as pg
    st = pg.TrainState(pg.init_model(pg.HyperParams(**HYP), seed=0), _image(),
                       pg.TrainConfig(batch_size=2 * B_LOCAL, seed=0), exact_mlp=True)
    loss = st.step()
    a = np.load(os.path.join(dp_run, "step1_rank0.npz"))
    assert abs(float(a["loss"]) - loss) <= 1e-6 * loss
    np.testing.assert_allclose(a["dense"], st.model.dense.cpu().numpy(), rtol=1e-5, atol=1e-7)
    # confidences: Adam on ~zero gradients (see test_train_step_parity_c1)
    conf = st.model.conf.cpu().numpy()
    assert (np.abs(a["conf"] - conf) > 1e-7 + 1e-5 * np.abs(conf)).mean() <= 0.002
    assert (a["baked"] != st.model.baked.cpu().numpy()).mean() <= 0.0005


class _SoloDist:
    """world-1 stand-in for torch.distributed (the all-reduce is the identity)."""
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


def test_dataparallel_divergence_raises_and_keeps_step_count():
    """DataParallel.step applies TrainState's divergence rule: a non-finite
    global loss raises TrainingDiverged, the optimizer kernels skipped the
    update and the step count is not advanced (trainer.py:131-133)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2312_17241_b200 as pg
    from paper_2312_17241_b200.dist import DataParallel
    kw = dict(n_f=32, n_c=64, n_p=4, n_levels=3, n_min=4, n_max=16, n_neurons=8)
    img = np.random.default_rng(2).random((12, 12, 3)).astype(np.float32)
    st = pg.TrainState(pg.init_model(pg.HyperParams(**kw), seed=0), img,
                       pg.TrainConfig(batch_size=64, lr=1e25, seed=0))
    dp = DataParallel(st, _SoloDist)
    with pytest.raises(pg.TrainingDiverged):
        for _ in range(50):
            t0 = st.t
            before = st.model.dense.clone()
            dp.step()
    assert st.t == t0
    assert torch.equal(st.model.dense, before)
