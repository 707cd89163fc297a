"""Config-1 (B=100) and config-2 small-layer timings of smb_spmm / smb_spmm_t
with the W=1 ring depth forced by SMB_SPMM_W (11: U=8, 12: U=16, 1: U=32)."""
import os, sys; sys.path.insert(0, '.')
import torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01))
def timeit(f, reps=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(5_000_000)
    s.record()
    for _ in range(reps): f()
    e.record(); e.synchronize()
    return s.elapsed_time(e) * 1e3 / reps
out = []
for B in (100, 1024):
    for li, layer in enumerate(model.layers):
        if not isinstance(layer, smb.SparseLinearLayer):
            continue
        W = layer.weights; m, k = W.nrows, W.ncols
        if B == 1024 and m != 10:
            continue
        x = torch.rand(k, B, device="cuda"); y = torch.empty(m, B, device="cuda")
        d = torch.randn(m, B, device="cuda"); dx = torch.empty(k, B, device="cuda")
        mask = torch.rand(k, B, device="cuda") - 0.3; bias = torch.zeros(m, device="cuda")
        f = lambda: _lib.call("smb_spmm", 0, ptr(W.row_ptr), ptr(W.col_idx), ptr(W.values), m, k,
                              ptr(x), B, B, ptr(bias), 1, ptr(y), B, stream_ptr())
        g = lambda: _lib.call("smb_spmm_t", 0, W.pattern.handle, ptr(W.values), ptr(d), B, B,
                              ptr(mask), B, ptr(dx), B, stream_ptr())
        out.append(f"B={B} L{li} {m}x{k}: fwd {timeit(f):.2f} T {timeit(g):.2f}")
print("W", os.environ.get("SMB_SPMM_W", "auto"), " | ".join(out))
