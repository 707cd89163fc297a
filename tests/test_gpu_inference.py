"""Batch-1 / small-batch inference (bench.py:366-399):
the graph-captured InferenceSession equals Sequential.feedforward bit for bit
(sparse and masked backends, saturated dense last layer included) and the
oracle's forward (bit-exact on all-sparse chains)."""

import numpy as np
import pytest

from conftest import bits_equal

pytestmark = pytest.mark.gpu

import paper_2407_17437_b200 as smb  # noqa: E402


@pytest.mark.parametrize("backend,density", [("sparse", 0.01), ("sparse", 0.1),
                                             ("masked", 0.01)])
@pytest.mark.parametrize("batch", [1, 7])
def test_session_equals_feedforward(backend, density, batch):
    cfg = smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=density, seed=8,
                               backend=backend)
    model, _ = smb.build_model(cfg)
    model.eval_mode()
    sess = smb.InferenceSession(model, batch=batch)
    rng = np.random.default_rng(batch)
    for _ in range(3):  # first call captures, later calls replay with new inputs
        x = rng.standard_normal((3072, batch)).astype(np.float32)
        got = sess(x)
        want = smb.to_numpy(model.feedforward(x))
        assert got.shape == (10, batch)
        assert bits_equal(got, want)


def test_session_matches_oracle_forward(oracle):
    chain = [3072, 1024, 512, 10]
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=chain, density=0.01, seed=4))
    ref = oracle.OracleMLP.build(chain, 0.01, seed=4)
    assert all(l.sparse for l in ref.layers)
    x = np.random.default_rng(0).standard_normal((3072, 1)).astype(np.float32)
    got = smb.InferenceSession(model, batch=1)(x)
    assert bits_equal(got, ref.forward(x))


def test_bench_inference_reports_reference_keys():
    cfg = smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01, seed=0)
    r = smb.bench_inference(cfg, n_repeats=20, warmup=3)
    assert set(r) == {"backend", "density", "layer_dims", "repeats", "mean_ms", "median_ms",
                      "min_ms", "max_ms"}
    assert r["repeats"] == 20 and 0 < r["min_ms"] <= r["median_ms"] <= r["max_ms"]
    with pytest.raises(smb.InvalidArgumentError):
        smb.bench_inference(cfg, n_repeats=0)
