"""Multi-GPU: data-parallel training with ONE all-reduce per step, and
query-sharded inference.  One process per GPU; the collective is
torch.distributed over NCCL on NVLink/NVSwitch (gloo works for the CPU tests).

Training step on every replica r of G:

    batch_r = slice r of the global batch          (independent sampling)
    compute_grads(batch_r)                         (loss grad scaled 2/(G*B*out))
    pack:   touched flags -> float slots, loss sum -> last slot
    all_reduce(SUM) over ONE flat buffer
            [gfeats | gmlp | pad | gconf | pad | touched | loss]
    unpack: touched = union of replicas' rows (a row any replica looked up is
            updated everywhere, so lazy Adam moves the same rows on every
            replica and replicas stay bit-identical), loss = global sum
    dense Adam + lazy Adam/re-bake, identical on every replica

The reference has no parallelism; the sum of the replicas'
gradients equals the single-process gradient of the concatenated batch up to
summation order, which tests/test_dist.py checks.
"""

from __future__ import annotations


class DataParallel:
    """Wraps a TrainState-like object (sample_batch / compute_grads /
    exchange_buffer / pack_exchange / unpack_exchange / apply_updates /
    loss_sum / t) and a torch.distributed-like module."""

    def __init__(self, state, dist, group=None):
        self.state, self.dist, self.group = state, dist, group
        self.rank = dist.get_rank(group) if group is not None else dist.get_rank()
        self.world = dist.get_world_size(group) if group is not None else dist.get_world_size()
        state.shard(self.rank, self.world)

    def launch_step(self) -> None:
        st = self.state
        xs, targets = st.sample_batch()
        st.loss_sum.zero_()
        st.compute_grads(xs, targets)
        st.pack_exchange()
        self.dist.all_reduce(st.exchange_buffer(), op=self.dist.ReduceOp.SUM, group=self.group)
        st.unpack_exchange()
        st.t += 1
        st.apply_updates()

    def step(self) -> float:
        """One data-parallel step; raises TrainingDiverged (and keeps the
        step count) on a non-finite global loss, like TrainState.step."""
        self.launch_step()
        return self.state.finish_step()


def shard_range(n: int, rank: int, world: int):
    """Contiguous [lo, hi) slice of n independent queries for one rank
    (rows are independent, model_io.py:294-295: no collective needed)."""
    per = (n + world - 1) // world
    lo = min(n, rank * per)
    return lo, min(n, lo + per)
