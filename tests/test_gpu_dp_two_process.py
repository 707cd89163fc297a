"""The engine's data-parallel step at world size 2.

Two processes share cuda:0 over a gloo process group (gloo all-reduces CUDA
tensors through the host, so no kernel of one rank waits on a kernel of the
other).  Each rank runs FusedTrainStep(process_group=...) on its B/2 slice of
every global batch (shard_epoch), scales the loss gradient by 1/B_global and
sums each layer's [values | bias] bucket with an all-reduce right after that
layer's gradients exist, then applies the update -- the code path bench.py
runs over NCCL on N GPUs.  The replicas must stay bit-identical and match the
single-process fused step at the global batch within 1e-5 (only the order of
the batch reduction differs).  Reference loop: train.py:389-402, /B at :399.
"""

import os
import socket

import numpy as np
import pytest
import torch

from conftest import bits_equal, rel_err

pytestmark = pytest.mark.gpu

CHAIN, DENS, SEED, B_GLOBAL, WORLD, STEPS, ETA = [3072, 1024, 512, 10], 0.01, 3, 256, 2, 4, 0.02


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    import paper_2407_17437_b200 as smb

    return smb.synthetic_dataset(seed=13, n_samples=B_GLOBAL * STEPS, features=CHAIN[0])


def _worker(rank, port, outdir, chain, density, bucketed):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import paper_2407_17437_b200 as smb

    data = _data()
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=density,
                                                    seed=SEED, batch_size=B_GLOBAL, lr=ETA))
    b_local = B_GLOBAL // WORLD
    step = smb.FusedTrainStep(model, b_local, global_batch=B_GLOBAL,
                              process_group=dist.group.WORLD, bucketed=bucketed)
    assert step.dp and step.world == WORLD and not step.graph_comm
    step.attach_dataset(smb.DeviceDataset(data))
    perm = np.random.default_rng(7).permutation(B_GLOBAL * STEPS)
    step.set_epoch(perm, rank_offset=rank * b_local)
    losses = []
    for _ in range(STEPS):
        step.step(ETA)
        losses.append(step.loss_value())
    torch.cuda.synchronize()
    params = {n: t.detach().cpu().numpy().reshape(-1) for n, t in model.parameters()}
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), losses=np.array(losses), **params)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("chain,density", [
    (CHAIN, 0.01),
    ([3072, 1024, 512, 10], 0.1),  # dense (ER-saturated) output layer
])
@pytest.mark.parametrize("bucketed", [True, False])
def test_two_rank_engine_matches_global_batch(tmp_path, chain, density, bucketed):
    import torch.multiprocessing as mp

    import paper_2407_17437_b200 as smb

    mp.start_processes(_worker, args=(_free_port(), str(tmp_path), chain, density, bucketed),
                       nprocs=WORLD, join=True, start_method="spawn")
    ranks = [np.load(tmp_path / f"rank{r}.npz") for r in range(WORLD)]
    names = [n for n in ranks[0].files if n != "losses"]
    for n in names:  # replicas stay bit-identical
        assert bits_equal(ranks[0][n], ranks[1][n]), n
    # single process, global batch, the plain fused step
    data = _data()
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=density,
                                                    seed=SEED, batch_size=B_GLOBAL, lr=ETA))
    step = smb.FusedTrainStep(model, B_GLOBAL)
    step.attach_dataset(smb.DeviceDataset(data))
    step.set_epoch(np.random.default_rng(7).permutation(B_GLOBAL * STEPS))
    total = []
    for _ in range(STEPS):
        step.step(ETA)
        total.append(step.loss_value())
    torch.cuda.synchronize()
    # the two ranks' local losses add up to the global batch loss
    assert np.allclose(ranks[0]["losses"] + ranks[1]["losses"], total, rtol=1e-5)
    for n, t in model.parameters():
        err = rel_err(ranks[0][n], t.detach().cpu().numpy().reshape(-1))
        assert err <= 1e-5, (n, err)


def _nccl_worker(rank, port, outdir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    import paper_2407_17437_b200 as smb

    data = _data()
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=CHAIN, density=DENS, seed=SEED,
                                                    batch_size=B_GLOBAL, lr=ETA))
    # (a world of one runs the single-GPU step unless the data-parallel
    # structure is forced -- bench.py --force-dp does the same)
    step = smb.FusedTrainStep(model, B_GLOBAL, process_group=dist.group.WORLD, force_dp=True)
    assert step.dp and step.bucketed and step.graph_comm and step.use_graph
    step.attach_dataset(smb.DeviceDataset(data))
    step.set_epoch(np.random.default_rng(7).permutation(B_GLOBAL * STEPS))
    for _ in range(STEPS):
        step.step(ETA)  # from the 2nd step on: graph replays with the captured NCCL buckets
    torch.cuda.synchronize()
    params = {n: t.detach().cpu().numpy().reshape(-1) for n, t in model.parameters()}
    np.savez(os.path.join(outdir, "nccl.npz"), **params)
    dist.destroy_process_group()


def test_nccl_world_of_one_graph_captured_buckets_equal_fused(tmp_path):
    """The per-layer NCCL all-reduce buckets captured into the step's CUDA
    graph (the bench's multi-GPU path), run over a world of one: the
    collectives are the identity, so the parameters must equal the plain
    fused single-GPU step bit for bit -- the capture, the stream joins and the
    per-layer update placement are exercised exactly as at N GPUs."""
    import torch.multiprocessing as mp

    import paper_2407_17437_b200 as smb

    mp.start_processes(_nccl_worker, args=(_free_port(), str(tmp_path)), nprocs=1, join=True,
                       start_method="spawn")
    got = np.load(tmp_path / "nccl.npz")
    data = _data()
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=CHAIN, density=DENS, seed=SEED,
                                                    batch_size=B_GLOBAL, lr=ETA))
    step = smb.FusedTrainStep(model, B_GLOBAL)
    step.attach_dataset(smb.DeviceDataset(data))
    step.set_epoch(np.random.default_rng(7).permutation(B_GLOBAL * STEPS))
    for _ in range(STEPS):
        step.step(ETA)
    torch.cuda.synchronize()
    for n, t in model.parameters():
        assert bits_equal(got[n], t.detach().cpu().numpy().reshape(-1)), n


def _sgd_worker(rank, port, outdir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    import paper_2407_17437_b200 as smb

    cfg = smb.ExperimentConfig(layer_dims=CHAIN, density=DENS, seed=SEED, batch_size=B_GLOBAL,
                               lr=ETA, epochs=2, eval_metrics=False, world_size=WORLD)
    model, _ = smb.build_model(cfg)
    recs = smb.sgd_train(model, _data(), smb.TrainConfig(epochs=2, batch_size=B_GLOBAL,
                                                         schedule=cfg.schedule(),
                                                         eval_metrics=False),
                         process_group=dist.group.WORLD)
    assert len(recs) == 2
    torch.cuda.synchronize()
    np.savez(os.path.join(outdir, f"sgd{rank}.npz"),
             **{n: t.detach().cpu().numpy().reshape(-1) for n, t in model.parameters()})
    dist.barrier()
    dist.destroy_process_group()


def test_sgd_train_data_parallel_matches_single_process(tmp_path):
    """sgd_train(process_group=...) with ExperimentConfig(world_size=2): the
    drop-in training loop (train.py:357-423) sharded over two ranks equals the
    single-process run at the same global batch within 1e-5, replicas
    bit-identical."""
    import torch.multiprocessing as mp

    import paper_2407_17437_b200 as smb

    mp.start_processes(_sgd_worker, args=(_free_port(), str(tmp_path)), nprocs=WORLD, join=True,
                       start_method="spawn")
    ranks = [np.load(tmp_path / f"sgd{r}.npz") for r in range(WORLD)]
    for n in ranks[0].files:
        assert bits_equal(ranks[0][n], ranks[1][n]), n
    cfg = smb.ExperimentConfig(layer_dims=CHAIN, density=DENS, seed=SEED, batch_size=B_GLOBAL,
                               lr=ETA, epochs=2, eval_metrics=False)
    model, _ = smb.build_model(cfg)
    smb.sgd_train(model, _data(), smb.TrainConfig(epochs=2, batch_size=B_GLOBAL,
                                                  schedule=cfg.schedule(), eval_metrics=False))
    torch.cuda.synchronize()
    for n, t in model.parameters():
        err = rel_err(ranks[0][n], t.detach().cpu().numpy().reshape(-1))
        assert err <= 1e-5, (n, err)
