"""Data-parallel plumbing of the pruned RNN-T loss: the batch shards by
utterance, one process per GPU; the only exchange of a step is the sum over ranks of the joiner-weight
gradients d_w (V,J), d_b (V) and of the two batch losses.  They live in ONE flat fp32 buffer

    flat = [ d_w (V*J) | d_b (V) | loss sums (2) ]

whose views are the step's d_w / d_b outputs.  How each rank's contribution reaches it is the
library's rnnt_exchange_mode_t (include/rnnt.h); the arithmetic (split-K reduction, loss combination
with infeasible utterances masked) runs in the library's kernels, this module only allocates,
zeroes, synchronises and calls torch.distributed:

* ``"nccl"`` (STORE): the kernels store this rank's values, then one all_reduce over ``flat``.
* ``"multimem"`` (MULTIMEM, NVLS): ``flat`` is torch symmetric memory; the kernels add into its
  multicast address with ``multimem.red.add``, so the NVSwitch sums over ranks and there is no
  separate all_reduce pass.  Zero -> barrier -> adds -> barrier.
* ``"red"`` (RED): several shards (or launches) add into one zeroed device buffer
  (``red.global.add``) -- the single-GPU form, parity-tested on one device.
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
    """The flat exchange buffer of one step and the way it is reduced across ranks.

    ``mode``: "nccl" (plain stores + all_reduce), "multimem" (NVLS multicast adds into symmetric
    memory), "red" (adds into one zeroed local buffer), or "local" (plain stores, no exchange)."""

    MODES = {"local": 0, "nccl": 0, "red": 1, "multimem": 2}

    def __init__(self, V: int, J: int, device, mode: str = "nccl", group=None):
        if mode not in self.MODES:
            raise ValueError(f"unknown exchange mode {mode!r}")
        self.V, self.J, self.mode, self.group = V, J, mode, group
        self.lib_mode = self.MODES[mode]
        self.zero_on_begin = True       # False: the caller zeroes once and several steps add (RED)
        n = self.flat_size(V, J)
        self.handle = None
        if mode == "multimem":
            import torch.distributed._symmetric_memory as symm_mem
            self.flat = symm_mem.empty(n, dtype=torch.float32, device=device)
            grp = group if group is not None else dist.group.WORLD
            self.handle = symm_mem.rendezvous(self.flat, grp)
            mc = int(self.handle.multicast_ptr)
            if mc == 0:
                raise RuntimeError("no NVLS multicast support on this device / group")
            self.addr_base = mc
        else:
            self.flat = torch.zeros(n, dtype=torch.float32, device=device)
            self.addr_base = None
        self.d_w = self.flat[: V * J].view(V, J)
        self.d_b = self.flat[V * J: V * J + V]
        self.loss_sums = self.flat[V * J + V: V * J + V + 2]

    @staticmethod
    def flat_size(V: int, J: int) -> int:
        """V*J + V + 2 floats rounded up to a multiple of 4 (16-B aligned rows when stacked)."""
        return (V * J + V + 2 + 3) // 4 * 4

    @classmethod
    def view_of(cls, flat: torch.Tensor, V: int, J: int):
        """A "local" (plain stores) buffer over an existing flat tensor of V*J + V + 2 floats (one row
        of a grouped step's partials)."""
        self = cls.__new__(cls)
        self.V, self.J, self.mode, self.group = V, J, "local", None
        self.lib_mode, self.zero_on_begin, self.handle, self.addr_base = 0, True, None, None
        self.flat = flat
        self.d_w = flat[: V * J].view(V, J)
        self.d_b = flat[V * J: V * J + V]
        self.loss_sums = flat[V * J + V: V * J + V + 2]
        return self

    # device addresses the kernels write / add to (multicast addresses in "multimem" mode)
    def target(self, which: str):
        if self.addr_base is None:
            return {"d_w": self.d_w, "d_b": self.d_b, "loss_sums": self.loss_sums}[which]
        off = {"d_w": 0, "d_b": self.V * self.J, "loss_sums": self.V * self.J + self.V}[which]
        return self.addr_base + 4 * off

    def begin(self, stream=None):
        """Before the step's adds: zero the buffer (all adding modes) and, for multimem, make sure
        every rank has zeroed its copy before any rank adds into it."""
        if self.lib_mode == 0 or not self.zero_on_begin:
            return
        with torch.cuda.stream(stream) if stream is not None else _null():
            self.flat.zero_()
            if self.handle is not None:
                self.handle.barrier(channel=0)

    def finish(self, stream=None, async_op: bool = False):
        """After the step's contributions: make the sum over ranks visible in ``flat``."""
        if self.mode == "nccl":
            return allreduce_grads(self, self.group, async_op)
        if self.handle is not None:
            with torch.cuda.stream(stream) if stream is not None else _null():
                self.handle.barrier(channel=0)
        return None


class _null:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


def allreduce_grads(buf: GradBuffer, group=None, async_op: bool = False):
    """Sum d_w, d_b and the loss sums over the process group (one collective)."""
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(buf.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)
