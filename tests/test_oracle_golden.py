"""The CPU oracle (oracle/) against the reference's own outputs (tests/golden/,
written by tests/golden/make_golden.py from /root/reference in the build
container) -- the pin that makes the oracle a valid checker for the GPU path.
CPU only."""

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, bits_equal

K = np.load(GOLDEN / "kernels.npz")
PI = json.loads((GOLDEN / "plans_init.json").read_text())


def cases():
    return range(int(K["ncases"][0]))


@pytest.mark.parametrize("c", cases())
def test_kernels_bit_exact_vs_reference(oracle, c):
    p = f"c{c:03d}_"
    m, k, n = (int(v) for v in K[p + "shape"])
    rp, ci, v = K[p + "row_ptr"], K[p + "col_idx"], K[p + "values"]
    assert bits_equal(oracle.spmm(rp, ci, v, K[p + "x"]), K[p + "spmm"])
    for nb in (1, 3, 8):  # result independent of the block split
        assert bits_equal(oracle.spmm_t(rp, ci, v, k, K[p + "d"], nblocks=min(nb, max(k, 1))),
                          K[p + "spmm_t"])
    assert bits_equal(oracle.sddmm(rp, ci, K[p + "a"], K[p + "b"]), K[p + "sddmm"])
    s = v.copy()
    alpha, beta = K[p + "ab"]
    oracle.axpby(alpha, s, beta, K[p + "t"])
    assert bits_equal(s, K[p + "combine"])


def test_empty_pattern(oracle):
    out = oracle.spmm(np.zeros(5, np.int32), np.zeros(0, np.int32), np.zeros(0, np.float32),
                      np.ones((3, 6), np.float32))
    assert bits_equal(out, K["empty_spmm"])


def test_optimizer_trajectories_bit_exact(oracle):
    O = np.load(GOLDEN / "optimizer.npz")
    for name, mu, nesterov in (("gd", 0.0, False), ("mom", 0.9, False), ("nesterov", 0.9, True)):
        lay = oracle.Layer(7, 6, False, True, O["values0"], O["row_ptr"], O["col_idx"], mu, nesterov)
        ref = oracle.OracleMLP([lay])
        for s in range(10):
            if name == "gd":  # GradientDescent: w += f(-eta) g (nn.py:196-197)
                oracle.axpby(1.0, lay.values, -0.05, O["grads"][s])
                lay.bias += np.float32(-0.05) * O["gbias"][s]
            else:
                ref.optimize([(O["grads"][s], O["gbias"][s])], 0.05)
            assert bits_equal(lay.values, O[name + "_values"][s]), (name, s)
            assert bits_equal(lay.bias, O[name + "_bias"][s]), (name, s)


def test_er_plans_match_reference(oracle):
    for p in PI["plans"]:
        dens, nnz = oracle.er_plan(p["chain"], p["density"])
        assert nnz == p["layer_nnz"]
        assert dens == p["layer_densities"]


def test_initial_models_match_reference(oracle):
    for rec in PI["init"]:
        m = oracle.OracleMLP.build(rec["chain"], rec["density"], seed=rec["seed"])
        got = [(n, hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest())
               for n, a in m.parameters()]
        assert got == [(q["name"], q["sha256"]) for q in rec["params"]]
        pats = [{"row_ptr": hashlib.sha256(l.row_ptr.tobytes()).hexdigest(),
                 "col_idx": hashlib.sha256(l.col_idx.tobytes()).hexdigest()}
                for l in m.layers if l.sparse]
        assert pats == rec["patterns"]
        assert m.fingerprint() == rec["fingerprint"]


def test_train_trace_bit_exact(oracle):
    """12 reference training steps reproduced bit for bit (losses and every
    parameter) -- kernels, softmax-CE, bias, ReLU and Nesterov arithmetic."""
    from paper_2407_17437_b200.data import synthetic_dataset

    T = np.load(GOLDEN / "train_trace.npz")
    data = synthetic_dataset(seed=5, n_samples=1200, features=3072)
    m = oracle.OracleMLP.build([3072, 1024, 512, 10], 0.01, seed=0)
    for k in range(12):
        b = T["order"][k * 100:(k + 1) * 100]
        loss = m.step(data.Xtrain[:, b], data.Ttrain[:, b], 0.01)
        assert loss == T["losses"][k]
    for name, arr in m.parameters():
        assert bits_equal(arr, T["p_" + name]), name
    assert m.fingerprint() == str(T["fingerprint"])


def test_reference_recorded_fingerprint(oracle):
    """pkg/test_output.txt:26 (criterion 7): the oracle reproduces the
    reference's recorded SHA-256 weight fingerprint of a 10-step run."""
    fp = json.loads((GOLDEN / "fingerprints.json").read_text())
    xtr, ttr, _, _ = oracle.synthetic_blobs(10, 3072, 50, 1.0, 3, 5)
    m = oracle.OracleMLP.build([3072, 1024, 512, 10], 0.01, seed=3)
    m.train(xtr, ttr, 2, 100, oracle.multistep(0.1))
    assert m.fingerprint() == fp["sparse_seed3_2epochs_B100_blobs50"]
    assert m.fingerprint().startswith(fp["recorded_prefix_test_output_txt_26"])


def test_reference_recorded_masked_fingerprint(oracle):
    """The masked-dense baseline (MaskedDense, train.py:159-170; nn.py:201-264)
    of the same run reproduces the recorded masked fingerprint
    (pkg/test_output.txt:26, cb8714b95a57...)."""
    fp = json.loads((GOLDEN / "fingerprints.json").read_text())
    xtr, ttr, _, _ = oracle.synthetic_blobs(10, 3072, 50, 1.0, 3, 5)
    m = oracle.OracleMLP.build([3072, 1024, 512, 10], 0.01, seed=3, backend="masked")
    m.train(xtr, ttr, 2, 100, oracle.multistep(0.1))
    assert m.fingerprint() == fp["masked_seed3_2epochs_B100_blobs50"]
    assert m.fingerprint().startswith(fp["recorded_prefix_masked_test_output_txt_26"])


def test_pcg64_restatement_matches_numpy(oracle):
    """The device Xavier kernel's algorithm (PCG64 XSL-RR + LCG jump-ahead)
    against numpy's own generator and xavier_init's float64->fp32 mapping."""
    for seed, key in ((3, 1), (0, 1), (123, 4)):
        seq = np.random.SeedSequence(entropy=seed, spawn_key=(key,))
        g = np.random.Generator(np.random.PCG64(seq))
        st = g.bit_generator.state["state"]
        a = float(np.sqrt(6.0 / (3072 + 1024)))
        want = g.uniform(-a, a, size=40).astype(np.float32)
        for off in (0, 7, 31):
            got = oracle.pcg_uniform(st["state"], st["inc"], off, 40 - off, a).astype(np.float32)
            assert bits_equal(got, want[off:])
        g2 = np.random.Generator(np.random.PCG64(seq))
        raw = g2.bit_generator.random_raw(5)
        s = st["state"]
        for r in raw:
            s = (s * oracle.PCG_MULT + st["inc"]) & oracle.M128
            assert oracle.pcg_output(s) == int(r)
