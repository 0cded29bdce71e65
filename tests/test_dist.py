"""N > 1 data-parallel host logic on CPU (world size 2, gloo): each rank takes its shard of a
global batch (dist.shard_indices), computes its joiner-weight gradients and loss sums (here with
the fp64 oracle, standing in for the CUDA path which needs a GPU), writes them into a GradBuffer
and all_reduces; the result must equal the oracle over the whole global batch."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_batch():
    return synth.make_custom([9, 6, 12, 7, 5], [3, 2, 4, 2, 1], 16, 8, 3, seed=5, logit_scale=1.5)


def _rank_sums(b, idx):
    from paper_2206_13236_b200.dist import GradBuffer
    buf = GradBuffer(b.V, b.J, "cpu", mode="local")
    ls, lp = [], []
    for n in idx:
        d = b.utterance(int(n))
        s = O.simple_loss(d["am"], d["lm"], d["y"], 0.5)
        ls.append(s["loss"])
        p = O.adjust_bounds(O.raw_bounds(s["px_grad"], s["py_grad"], d["S"]), d["T"], d["U"], d["S"])
        r = O.pruned_loss(d["enc"], d["dec"], d["W"], d["b"], d["y"], p, d["S"], 1.0, matched=True)
        lp.append(r["loss"])
        buf.d_w += torch.from_numpy(r["d_w"]).float()
        buf.d_b += torch.from_numpy(r["d_b"]).float()
    # the loss combination of P:318-323 (on the GPU path: the library's rnnt_loss_sums)
    buf.loss_sums[0] = 0.5 * float(np.sum(ls))
    buf.loss_sums[1] = 1.0 * float(np.sum([x for x in lp if np.isfinite(x)]))
    return buf


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2206_13236_b200.dist import allreduce_grads, shard_indices
    b = _global_batch()
    idx = shard_indices(b.T_n, b.U_n, world, rank)
    buf = _rank_sums(b, idx)
    allreduce_grads(buf)
    out[rank] = (idx.tolist(), buf.flat.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_indices_partition_and_balance():
    from paper_2206_13236_b200.dist import shard_indices
    T = np.array([100, 400, 250, 300, 120, 90, 500])
    U = np.array([20, 100, 40, 90, 30, 10, 150])
    parts = [shard_indices(T, U, 3, r) for r in range(3)]
    allidx = np.sort(np.concatenate(parts))
    assert np.array_equal(allidx, np.arange(7))
    cost = T * (U + 1)
    loads = [cost[p].sum() for p in parts]
    assert max(loads) <= 2.0 * min(loads)


def test_allreduce_world2_matches_global_oracle():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    b = _global_batch()
    ref = _rank_sums(b, np.arange(b.N)).flat.numpy()
    shards = sorted(i for r in range(world) for i in res[r][0])
    assert shards == list(range(b.N))
    for r in range(world):
        got = res[r][1]
        assert np.allclose(got, ref, rtol=1e-5, atol=1e-5), np.abs(got - ref).max()
