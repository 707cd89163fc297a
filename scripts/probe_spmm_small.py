"""Time smb_spmm / smb_spmm_t on the config-2 layers (B=1024, warm L2, GPU held).
SMB_SPMM_W forces the lane width (1, 4, 8)."""
import os, sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
B = 1024
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01,
                                                batch_size=B, lr=0.01))
out = []
def timeit(f, reps=50):
    for _ in range(5): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(5_000_000)
    s.record()
    for _ in range(reps): f()
    e.record(); e.synchronize()
    return s.elapsed_time(e) * 1e3 / reps
for li, layer in enumerate(model.layers):
    if not hasattr(layer, "weights") or not isinstance(layer, smb.SparseLinearLayer):
        continue
    W = layer.weights
    m, k = W.nrows, W.ncols
    x = torch.rand(k, B, device="cuda"); y = torch.empty(m, B, device="cuda")
    d = torch.randn(m, B, device="cuda"); dx = torch.empty(k, B, device="cuda")
    mask = torch.rand(k, B, device="cuda") - 0.3
    bias = torch.zeros(m, device="cuda")
    f = lambda: _lib.call("smb_spmm_p", 0, W.pattern.handle, ptr(W.values), ptr(x), B, B,
                          ptr(bias), 1, ptr(y), B, stream_ptr())
    g = lambda: _lib.call("smb_spmm_t", 0, W.pattern.handle, ptr(W.values), ptr(d), B, B,
                          ptr(mask), B, ptr(dx), B, stream_ptr())
    out.append(f"L{li} {m}x{k} z={W.nnz}: fwd {timeit(f):.2f} us, T {timeit(g):.2f} us")
print("W", os.environ.get("SMB_SPMM_W", "auto"), " | ".join(out))
