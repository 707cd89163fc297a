"""Model archive I/O (data_io.py:250-535).

CPU: NPY / manifest validation paths (no device needed).
GPU: archives written by the reference itself (tests/golden/archive_*, made by
tests/golden/make_golden.py) load bit-identically; saving them again writes
byte-identical files; a trained device model round-trips.
"""

import json
import shutil
from pathlib import Path

import numpy as np
import pytest

import paper_2407_17437_b200 as smb

GOLDEN = Path(__file__).resolve().parent / "golden"


# ---------------------------------------------------------------- CPU ------
def test_save_npy_rejects_unsupported_dtype(tmp_path):
    with pytest.raises(smb.InvalidArgumentError):
        smb.save_npy(tmp_path / "a.npy", np.zeros(3, np.int64))
    smb.save_npy(tmp_path / "b.npy", np.arange(3, dtype=np.int32))
    assert smb.load_npy(tmp_path / "b.npy", np.int32, (3,)).tolist() == [0, 1, 2]


def test_load_npy_validation(tmp_path):
    with pytest.raises(smb.DatasetIOError):
        smb.load_npy(tmp_path / "missing.npy")
    bad = tmp_path / "bad.npy"
    bad.write_bytes(b"NOTNPY" + b"\0" * 64)
    with pytest.raises(smb.FormatError, match="magic"):
        smb.load_npy(bad)
    corrupt = tmp_path / "corrupt.npy"
    corrupt.write_bytes(b"\x93NUMPY\x01\x00\xff\xff garbage")
    with pytest.raises(smb.FormatError):
        smb.load_npy(corrupt)
    smb.save_npy(tmp_path / "f.npy", np.zeros((2, 3), np.float32))
    with pytest.raises(smb.FormatError, match="dtype"):
        smb.load_npy(tmp_path / "f.npy", np.float64)
    with pytest.raises(smb.FormatError, match="shape"):
        smb.load_npy(tmp_path / "f.npy", np.float32, (3, 2))


def test_load_model_manifest_errors(tmp_path):
    with pytest.raises(smb.DatasetIOError, match="manifest"):
        smb.load_model(tmp_path)
    (tmp_path / "manifest.json").write_text("{not json")
    with pytest.raises(smb.FormatError, match="invalid JSON"):
        smb.load_model(tmp_path)
    (tmp_path / "manifest.json").write_text(json.dumps({"schema_version": "2.0", "dtype": "float32"}))
    with pytest.raises(smb.FormatError, match="schema version"):
        smb.load_model(tmp_path)


def test_reference_archive_weight_file_bytes():
    meta = json.loads((GOLDEN / "archives.json").read_text())
    for backend in ("sparse", "masked"):
        assert smb.archive_weight_file_bytes(GOLDEN / f"archive_{backend}") == \
            meta[backend]["weight_file_bytes"]


# ---------------------------------------------------------------- GPU ------
@pytest.mark.gpu
@pytest.mark.parametrize("backend", ["sparse", "masked"])
def test_reference_archive_loads_bit_identically(backend, tmp_path):
    meta = json.loads((GOLDEN / "archives.json").read_text())[backend]
    src = GOLDEN / f"archive_{backend}"
    model = smb.load_model(src)
    assert smb.weights_fingerprint(model) == meta["fingerprint"]
    assert smb.model_size_report(model).to_dict() == meta["size_report"]
    # forward on the same input as the reference (fp32, within 1e-5 of its sum)
    rng = np.random.default_rng(21)
    x = rng.standard_normal((64, 30)).astype(np.float32)
    y = model.feedforward(x)
    got = float(np.sum(smb.to_numpy(y), dtype=np.float64))
    assert abs(got - meta["forward_sum"]) <= 1e-5 * max(1.0, abs(meta["forward_sum"]))
    # saving again reproduces the reference's files byte for byte
    out = tmp_path / "again"
    smb.save_model(model, out)
    assert json.loads((out / "manifest.json").read_text()) == \
        json.loads((src / "manifest.json").read_text())
    for f in sorted(src.glob("*.npy")):
        assert (out / f.name).read_bytes() == f.read_bytes(), f.name


@pytest.mark.gpu
def test_trained_model_round_trip(tmp_path):
    cfg = smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01, seed=2,
                               batch_size=64, lr=0.02)
    model, _ = smb.build_model(cfg)
    data = smb.synthetic_dataset(seed=1, n_samples=256, features=3072)
    st = smb.FusedTrainStep(model, 64)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.arange(256))
    for _ in range(3):
        st.step(0.02)
    smb.save_model(model, tmp_path / "m")
    back = smb.load_model(tmp_path / "m")
    assert smb.weights_fingerprint(back) == smb.weights_fingerprint(model)
    # a corrupted structure is reported as a format error
    bad = tmp_path / "bad"
    shutil.copytree(tmp_path / "m", bad)
    ci = np.load(bad / "layer00_col_idx.npy")
    ci[1] = ci[0]  # duplicate column inside row 0
    np.save(bad / "layer00_col_idx.npy", ci)
    with pytest.raises(smb.FormatError, match="invalid CSR structure"):
        smb.load_model(bad)
