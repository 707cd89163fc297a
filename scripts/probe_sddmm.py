"""Time smb_sddmm_update on the three config-2 layers (B=1024, warm L2).
SMB_SDDMM_VARIANT selects the tile/chunk/stage variant (see sddmm.cu)."""
import os, sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr
B = 1024
model, _ = smb.build_model(smb.ExperimentConfig(layer_dims=[3072, 1024, 512, 10], density=0.01,
                                                batch_size=B, lr=0.01))
out = []
for li, layer in enumerate(model.layers):
    if not hasattr(layer, "weights"):
        continue
    W = layer.weights
    pat = W.pattern
    m, k = pat.nrows, pat.ncols
    d = torch.randn(m, B, device="cuda"); x = torch.randn(k, B, device="cuda")
    vals = W.values.clone(); vel = torch.zeros_like(vals)
    def f():
        _lib.call("smb_sddmm_update", 0, pat.handle, ptr(d), B, ptr(x), B, B, ptr(vals), ptr(vel),
                  None, None, None, None, 3, 0.9, 0.01, stream_ptr())
    for _ in range(5): f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(5_000_000)  # hold the GPU so the 50 launches queue up (no host gaps)
    s.record()
    for _ in range(50): f()
    e.record(); e.synchronize()
    us = s.elapsed_time(e) * 1e3 / 50
    out.append(f"L{li} {m}x{k} nnz={pat.nnz}: {us:.2f} us ({pat.nnz * B / us / 1e6:.2f} Tpairs/s)")
print("variant", os.environ.get("SMB_SDDMM_VARIANT", "0"), " | ".join(out))
