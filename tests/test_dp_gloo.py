"""Data-parallel algorithm of the fused step, exercised with world_size 2 over
gloo on the CPU (the GPU path runs the same host logic over NCCL):
each rank takes its shard_epoch() slice of every global batch, scales the loss
gradient by 1/B_global, packs value + bias gradients into one flat buffer
(flat_layout), all-reduces it (SUM) and applies the identical update.  Must
match the single-process full-batch step within 1e-5 and leave the replicas
bit-identical."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_17437_b200.engine import flat_layout, shard_epoch

CHAIN, DENS, SEED, B_LOCAL, WORLD, STEPS, ETA = [96, 64, 48, 10], 0.2, 4, 32, 2, 3, 0.05


def _data():
    rng = np.random.default_rng(1)
    n = WORLD * B_LOCAL * STEPS
    x = rng.standard_normal((CHAIN[0], n)).astype(np.float32)
    lab = rng.integers(0, CHAIN[-1], n)
    t = np.zeros((CHAIN[-1], n), np.float32)
    t[lab, np.arange(n)] = 1
    return x, t, np.random.default_rng(2).permutation(n)


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from oracle import oracle as O

    O.set_threads(1)
    x, t, perm = _data()
    m = O.OracleMLP.build(CHAIN, DENS, seed=SEED)
    idx, kb = shard_epoch(perm, WORLD * B_LOCAL, B_LOCAL, rank * B_LOCAL)
    layout, total = flat_layout([(l.n_out, l.values.shape[0]) for l in m.layers])
    for k in range(kb):
        b = idx[k * B_LOCAL:(k + 1) * B_LOCAL]
        y = m.forward(x[:, b])
        grads = m.backward(m.softmax_ce_grad(y, t[:, b]) / (WORLD * B_LOCAL))
        flat = np.zeros(total, np.float32)
        for (g, gb), (off, boff) in zip(grads, layout):
            flat[off:off + g.shape[0]] = g
            flat[boff:boff + gb.shape[0]] = gb
        ft = torch.from_numpy(flat)
        dist.all_reduce(ft)
        flat = ft.numpy()
        summed = [(flat[off:off + g.shape[0]].copy(), flat[boff:boff + gb.shape[0]].copy())
                  for (g, gb), (off, boff) in zip(grads, layout)]
        m.optimize(summed, ETA)
    out[rank] = [a.copy() for _, a in m.parameters()]
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_data_parallel_matches_full_batch(oracle):
    ctx = mp.get_context("spawn")
    with ctx.Manager() as man:
        out = man.dict()
        mp.start_processes(_worker, args=(_free_port(), out), nprocs=WORLD, join=True,
                           start_method="spawn")
        ranks = [out[r] for r in range(WORLD)]
    for a, b in zip(ranks[0], ranks[1]):  # replicas stay bit-identical
        assert a.tobytes() == b.tobytes()
    x, t, perm = _data()
    ref = oracle.OracleMLP.build(CHAIN, DENS, seed=SEED)
    G = WORLD * B_LOCAL
    for k in range(len(perm) // G):
        b = perm[k * G:(k + 1) * G]
        ref.step(x[:, b], t[:, b], ETA)
    for a, (_, e) in zip(ranks[0], ref.parameters()):
        err = np.max(np.abs(a.astype(np.float64) - e) / np.maximum(1.0, np.abs(e)))
        assert err <= 1e-5, err
