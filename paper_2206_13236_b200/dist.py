"""Data-parallel plumbing of the pruned RNN-T loss: the batch shards by
utterance, one process per GPU; the only exchange of a step is the sum of the joiner-weight
gradients d_w (V,J), d_b (V) and of the scalar losses, done as ONE all_reduce over a flat fp32
buffer whose views are the step's d_w / d_b outputs (NCCL over NVLink in bench.py; gloo in the
CPU tests).  Everything else (am/lm/enc/dec gradients, ranges) stays local to its rank.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard_indices(T_n, U_n, world: int, rank: int) -> np.ndarray:
    """Utterance indices of ``rank``'s shard: greedy longest-processing-time assignment of the
    utterances, by lattice cost T_n (U_n + 1), to the least-loaded rank (deterministic: ties go
    to the lower index / lower rank), so per-rank step times are balanced."""
    T_n = np.asarray(T_n, np.int64)
    U_n = np.asarray(U_n, np.int64)
    cost = T_n * (U_n + 1)
    order = sorted(range(len(T_n)), key=lambda i: (-int(cost[i]), i))
    load = [0] * world
    mine = []
    for i in order:
        r = min(range(world), key=lambda q: (load[q], q))
        load[r] += int(cost[i])
        if r == rank:
            mine.append(i)
    return np.array(sorted(mine), np.int64)


class GradBuffer:
    """One flat fp32 buffer holding d_w (V,J), d_b (V) and the two loss sums, so the whole
    exchange of a step is a single all_reduce (d_w / d_b are passed to the C-ABI as views)."""

    def __init__(self, V: int, J: int, device):
        self.V, self.J = V, J
        self.flat = torch.zeros(V * J + V + 2, dtype=torch.float32, device=device)
        self.d_w = self.flat[: V * J].view(V, J)
        self.d_b = self.flat[V * J: V * J + V]
        self.loss_sums = self.flat[V * J + V:]

    def set_losses(self, loss_simple: torch.Tensor, loss_pruned: torch.Tensor, simple_scale=0.5,
                   pruned_scale=1.0):
        """loss_sums = [simple_scale * sum_n loss_simple, pruned_scale * sum_n loss_pruned]."""
        torch.sum(loss_simple, dim=0, keepdim=True, out=self.loss_sums[0:1])
        torch.sum(loss_pruned, dim=0, keepdim=True, out=self.loss_sums[1:2])
        self.loss_sums[0:1].mul_(simple_scale)
        self.loss_sums[1:2].mul_(pruned_scale)


def allreduce_grads(buf: GradBuffer, group=None, async_op: bool = False):
    """Sum d_w, d_b and the loss sums over the process group (one collective)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(buf.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
