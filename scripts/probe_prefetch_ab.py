"""Config-2 step with the next batch's gather beside the chain kernel vs beside
the weight sides: back-to-back replays and replays with the L2 flush between."""
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
L, d, B = [3072, 1024, 512, 10], 0.01, 1024
data = smb.synthetic_dataset(seed=0, n_samples=50000, features=L[0], classes=L[-1])
dd = smb.DeviceDataset(data)
flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device="cuda")
for early in (False, True, False, True):
    model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=L, density=d, batch_size=B, lr=0.01))
    st = smb.FusedTrainStep(model, B); st.prefetch_beside_chain = early
    st.attach_dataset(dd); st.set_epoch(np.arange(data.Xtrain.shape[1]))
    for _ in range(6): st.step(0.01)
    torch.cuda.synchronize()
    b2b, fl = [], []
    for rep in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(40): st.step(0.01)
        e.record(); e.synchronize(); b2b.append(s.elapsed_time(e) * 1e3 / 40)
    for rep in range(30):
        flush.fill_(rep); flush.sum(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); st.step(0.01); e.record(); e.synchronize(); fl.append(s.elapsed_time(e) * 1e3)
    print("beside chain" if early else "at the end  ", "b2b", ["%.1f" % r for r in b2b], "flushed median %.1f" % float(np.median(fl)), flush=True)
