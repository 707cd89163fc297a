"""Generate the golden fixtures of tests/golden/ by running the REFERENCE
(pkg/src/sparsemlp, imported in place from /root/reference) in the build
container.  The fixtures pin the CPU oracle (oracle/) and, through it and
directly, the CUDA path.  /root/reference does not exist on the GPU box; only
the committed fixtures travel.

    python tests/golden/make_golden.py          # rewrites tests/golden/*
"""

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(HERE.parents[1]))

import sparsemlp as sm  # noqa: E402  (the reference)
from sparsemlp import nn as rnn  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def random_csr(rng, m, k, density, dtype, empty_rows):
    mask = rng.random((m, k)) < density
    if empty_rows and m > 2:
        mask[rng.choice(m, size=m // 3, replace=False)] = False
    dense = np.where(mask, rng.standard_normal((m, k)), 0.0).astype(dtype)
    return sm.csr_from_dense(dense)


def kernels():
    """Reference outputs of spmm / spmm_transposed / sddmm / sparse_combine on
    seeded random instances (tensor_core.py:227-306), fp32 and fp64, including
    empty rows, an empty pattern, n = 1 and odd n."""
    rng = np.random.default_rng(20241017)
    shapes = [(1, 1, 1), (3, 5, 2), (17, 13, 5), (40, 33, 37), (48, 40, 21), (33, 65, 1),
              (129, 20, 9)]
    out = {}
    case = 0
    for dtype in (np.float32, np.float64):
        for (m, k, n) in shapes:
            for density in (0.05, 0.3, 1.0):
                s = random_csr(rng, m, k, density, dtype, empty_rows=density < 1)
                x = rng.standard_normal((k, n)).astype(dtype)
                d = rng.standard_normal((m, n)).astype(dtype)
                a = rng.standard_normal((m, n)).astype(dtype)
                b = rng.standard_normal((k, n)).astype(dtype)
                t = rng.standard_normal(s.nnz).astype(dtype)
                alpha, beta = rng.uniform(-2, 2, size=2)
                comb = s.copy()
                sm.sparse_combine(alpha, comb, beta, s.pattern.with_values(t))
                p = f"c{case:03d}_"
                out.update({
                    p + "shape": np.array([m, k, n]), p + "row_ptr": s.row_ptr,
                    p + "col_idx": s.col_idx, p + "values": s.values, p + "x": x, p + "d": d,
                    p + "a": a, p + "b": b, p + "t": t, p + "ab": np.array([alpha, beta]),
                    p + "spmm": sm.spmm(s, x), p + "spmm_t": sm.spmm_transposed(s, d),
                    p + "sddmm": sm.sddmm(s.pattern, a, b).values, p + "combine": comb.values,
                })
                case += 1
    # empty pattern
    s = sm.SparsityPattern(4, 3, np.zeros(5, np.int32), np.zeros(0, np.int32)).zeros()
    x = rng.standard_normal((3, 6)).astype(np.float32)
    out["empty_spmm"] = sm.spmm(s, x)
    out["ncases"] = np.array([case])
    np.savez_compressed(HERE / "kernels.npz", **out)


def optimizer():
    """10 optimizer steps of SparseLinearLayer with fixed gradients
    (nn.py:187-198): values / velocity / bias after each step."""
    out = {}
    rng = np.random.default_rng(33)
    pattern = sm.csr_from_dense(np.where(rng.random((6, 7)) < 0.5, 1.0, 0.0).astype(np.float32)
                                + np.eye(6, 7, dtype=np.float32)).pattern
    values0 = rng.standard_normal(pattern.nnz).astype(np.float32)
    grads = rng.standard_normal((10, pattern.nnz)).astype(np.float32)
    gbias = rng.standard_normal((10, 6)).astype(np.float32)
    out["row_ptr"], out["col_idx"], out["values0"] = pattern.row_ptr, pattern.col_idx, values0
    out["grads"], out["gbias"] = grads, gbias
    for name, opt in (("gd", rnn.GradientDescent()), ("mom", rnn.Momentum(0.9)),
                      ("nesterov", rnn.Momentum(0.9, nesterov=True))):
        layer = rnn.SparseLinearLayer(pattern, values0.copy(), np.zeros(6, np.float32), opt)
        vals, biases = [], []
        for s in range(10):
            layer.grad.values[:] = grads[s]
            layer.grad_bias = gbias[s].copy()
            layer.optimize(0.05)
            vals.append(layer.weights.values.copy())
            biases.append(layer.bias.copy())
        out[name + "_values"] = np.stack(vals)
        out[name + "_bias"] = np.stack(biases)
    np.savez_compressed(HERE / "optimizer.npz", **out)


def plans_and_init():
    """ER plans of the BASELINE configs (sparsity.py:103-180) and hashes of the
    seeded initial model (patterns + Xavier values) of build_model."""
    chains = {"cfg1": [3072, 1024, 512, 10], "cfg4": [3072, 8192, 8192, 8192, 10],
              "cfg5": [3072, 65536, 65536, 10]}
    plans = []
    for name, dens_list in (("cfg1", [0.001, 0.005, 0.01, 0.05, 0.1, 0.2, 0.5, 1.0]),
                            ("cfg4", [0.01]), ("cfg5", [0.001])):
        for d in dens_list:
            p = sm.er_densities(chains[name], d)
            plans.append({"chain": chains[name], "density": d,
                          "layer_densities": p.layer_densities, "layer_nnz": p.layer_nnz})
    init = []
    for chain, d, seed in (([3072, 1024, 512, 10], 0.01, 3), ([3072, 1024, 512, 10], 0.1, 1),
                           ([100, 64, 64, 10], 0.3, 9)):
        model, _ = sm.build_model(sm.ExperimentConfig(layer_dims=chain, density=d, seed=seed))
        layers = []
        for name, arr in model.parameters():
            layers.append({"name": name, "sha256": sha(arr), "head": np.asarray(arr).reshape(-1)[:8].tolist()})
        pats = []
        for lay in model.layers:
            if isinstance(lay, rnn.SparseLinearLayer):
                pats.append({"row_ptr": sha(lay.weights.row_ptr), "col_idx": sha(lay.weights.col_idx)})
        init.append({"chain": chain, "density": d, "seed": seed, "params": layers,
                     "patterns": pats, "fingerprint": sm.weights_fingerprint(model)})
    (HERE / "plans_init.json").write_text(json.dumps({"plans": plans, "init": init}, indent=1))


def train_trace():
    """Per-step losses and final parameters of 12 reference steps (the loop body
    of train.py:398-401) at the config-1 shape, seed 0, lr 0.01, on the
    SURVEY.md 8(d) synthetic data (1,200 samples, B=100)."""
    from paper_2407_17437_b200.data import synthetic_dataset

    data = synthetic_dataset(seed=5, n_samples=1200, features=3072)
    model, _ = sm.build_model(sm.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01,
                                                  seed=0, lr=0.01))
    loss = rnn.SoftmaxCrossEntropyLoss()
    order = np.random.default_rng(7).permutation(1200)
    losses = []
    for k in range(12):
        b = order[k * 100:(k + 1) * 100]
        xb, tb = data.Xtrain[:, b], data.Ttrain[:, b]
        y = model.feedforward(xb)
        losses.append(rnn.softmax_ce_loss(y, tb))
        model.backpropagate(y, loss.gradient(y, tb) / 100)
        model.optimize(0.01)
    params = {f"p_{name}": np.asarray(a).copy() for name, a in model.parameters()}
    np.savez_compressed(HERE / "train_trace.npz", order=order, losses=np.array(losses),
                        fingerprint=np.array(sm.weights_fingerprint(model)), **params)


def fingerprints():
    """The runs behind pkg/test_output.txt:26 (criterion 7): sparse and
    masked backends, seed 3, 2 epochs, B=100, synthetic blobs 50/class."""
    out = {}
    for backend in ("sparse", "masked"):
        cfg = sm.ExperimentConfig(
            layer_dims=[3072, 1024, 512, 10], density=0.01, backend=backend, epochs=2,
            batch_size=100, seed=3, threads=1, eval_metrics=False,
            dataset="synthetic:classes=10,features=3072,per_class=50,spread=1.0,test_per_class=5")
        _, model = sm.run_training(cfg)
        out[f"{backend}_seed3_2epochs_B100_blobs50"] = sm.weights_fingerprint(model)
    recorded = (REF_SRC.parents[0] / "test_output.txt").read_text()
    out["recorded_prefix_test_output_txt_26"] = "69a2e92774f1" if "69a2e92774f1" in recorded else None
    out["recorded_prefix_masked_test_output_txt_26"] = (
        "cb8714b95a57" if "cb8714b95a57" in recorded else None)
    (HERE / "fingerprints.json").write_text(json.dumps(out, indent=1))


def archives():
    """Model archives written by the reference's save_model (data_io.py:359-380)
    for a small sparse and a small masked model after 3 training steps, plus
    their fingerprints / size reports: interop fixtures for archive.py."""
    from sparsemlp import data_io as dio

    rng = np.random.default_rng(21)
    x = rng.standard_normal((64, 30)).astype(np.float32)
    t = np.zeros((10, 30), np.float32)
    t[rng.integers(0, 10, 30), np.arange(30)] = 1
    meta = {}
    for backend in ("sparse", "masked"):
        model, _ = sm.build_model(sm.ExperimentConfig(
            layer_dims=[64, 48, 32, 10], density=0.2, seed=7, backend=backend, lr=0.05))
        loss = rnn.SoftmaxCrossEntropyLoss()
        for _ in range(3):
            y = model.feedforward(x)
            model.backpropagate(y, loss.gradient(y, t) / 30)
            model.optimize(0.05)
        d = HERE / f"archive_{backend}"
        dio.save_model(model, d)
        meta[backend] = {"fingerprint": sm.weights_fingerprint(model),
                         "size_report": dio.model_size_report(model).to_dict(),
                         "weight_file_bytes": dio.archive_weight_file_bytes(d),
                         "forward_sum": float(np.sum(model.feedforward(x), dtype=np.float64))}
    (HERE / "archives.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    sm.set_num_threads(1)
    kernels()
    optimizer()
    plans_and_init()
    train_trace()
    fingerprints()
    archives()
    for f in sorted(HERE.iterdir()):
        print(f.name, f.stat().st_size)
