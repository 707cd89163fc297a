"""Graph-timed per-kernel durations of the config-2 step (KernelTimer.
kernel_durations) under the library's tuning variables; one process per
setting (the library reads them once).  Usage:
  python scripts/probe_graph_variants.py            # runs every setting
  PGV_B=100 PGV_LAYERS=... python scripts/probe_graph_variants.py"""
import json, os, subprocess, sys
sys.path.insert(0, '.')

SETTINGS = [{}] + [{"SMB_SPMM_W": w} for w in ("1", "4", "7", "8", "9", "11", "12", "13", "14")] \
    + [{"SMB_SDDMM_VARIANT": v} for v in ("1", "2", "3")]


def child():
    import numpy as np, torch
    import paper_2407_17437_b200 as smb
    from paper_2407_17437_b200.engine import KernelTimer
    B = int(os.environ.get("PGV_B", "1024"))
    layers = [int(x) for x in os.environ.get("PGV_LAYERS", "3072,1024,512,10").split(",")]
    d = float(os.environ.get("PGV_D", "0.01"))
    data = smb.synthetic_dataset(seed=0, n_samples=4 * B, features=layers[0], classes=layers[-1])
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=layers, density=d, batch_size=B,
                                                    lr=0.01))
    st = smb.FusedTrainStep(model, B)
    st.attach_dataset(smb.DeviceDataset(data))
    st.set_epoch(np.arange(4 * B))
    for _ in range(3):
        st.step(0.01)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(300):
        st.step(0.01)
    e.record(); e.synchronize()
    out = KernelTimer().kernel_durations(st, 0.01)
    res = {t: round(1e3 * ms / c, 2) for t, (c, ms) in out.items()}
    res["step_b2b"] = round(s.elapsed_time(e) * 1e3 / 300, 2)
    print(json.dumps(res))


if __name__ == "__main__":
    if os.environ.get("PGV_CHILD") == "1":
        child()
        sys.exit(0)
    for env in SETTINGS:
        r = subprocess.run([sys.executable, __file__], env={**os.environ, **env, "PGV_CHILD": "1"},
                           capture_output=True, text=True, timeout=600)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(json.dumps(env), line, flush=True)
