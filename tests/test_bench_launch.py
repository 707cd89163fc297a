"""bench.py's multi-GPU launch logic (no GPU needed): `--gpus N` outside
torchrun re-runs the same command as N ranks through torch.distributed.run on
127.0.0.1; under torchrun (WORLD_SIZE set) or with N == 1 it runs in place;
the NCCL settings of the data-parallel runs are logged and pinned without
overriding a caller's choice."""

import importlib.util
import sys

import pytest

from conftest import REPO


@pytest.fixture()
def bench(monkeypatch):
    spec = importlib.util.spec_from_file_location("bench_under_test", REPO / "bench.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _args(bench, argv, monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py", *argv])
    return bench.parse_args()


def test_self_launch_spawns_n_ranks(bench, monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    args = _args(bench, ["--gpus", "4", "--steps", "7"], monkeypatch)
    assert bench.self_launch(args) == 0
    cmd = seen["cmd"]
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert "--master-addr=127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"]  # the same arguments, re-run per rank


@pytest.mark.parametrize("env,gpus", [({"WORLD_SIZE": "2"}, 2), ({}, 1)])
def test_no_relaunch_under_torchrun_or_single_gpu(bench, monkeypatch, env, gpus):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: pytest.fail("relaunched"))
    assert bench.self_launch(_args(bench, ["--gpus", str(gpus)], monkeypatch)) is None


def test_nccl_env_defaults_do_not_override(bench, monkeypatch):
    monkeypatch.delenv("NCCL_DEBUG", raising=False)
    monkeypatch.delenv("NCCL_DEBUG_SUBSYS", raising=False)
    monkeypatch.setenv("NCCL_ALGO", "Tree")
    bench.nccl_env()
    import os

    assert os.environ["NCCL_DEBUG"] == "INFO" and os.environ["NCCL_DEBUG_SUBSYS"] == "INIT"
    assert os.environ["NCCL_ALGO"] == "Tree"  # the caller's choice stands


def test_reference_arm_without_torchrun_uses_global_batch(bench, monkeypatch, capsys):
    """`--impl reference --gpus N` outside torchrun: one process times the CPU
    port on the N-rank global batch (rank 0's job under torchrun)."""
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: 0)  # (self_launch not used here)
    args = _args(bench, ["--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                         "--layers", "64,32,10", "--batch", "16"], monkeypatch)
    assert bench.run_reference(args) == 0
    import json

    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["global_batch"] == 32
    assert line["e2e"]["h2d_bytes_per_step"] == 0
