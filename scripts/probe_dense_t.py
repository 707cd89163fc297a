"""Time smb_dense_backward_input alone at the config-5 output-layer shapes
(W 10 x 65536, d 10 x B, mask / out 65536 x B) and list the kernel it ran."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2407_17437_b200 import _lib

k, m = 65536, 10
for B in (512, 4096):
    w = torch.randn(m, k, device="cuda")
    d = torch.randn(m, B, device="cuda")
    mk = torch.randn(k, B, device="cuda")
    out = torch.empty(k, B, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: _lib.call("smb_dense_backward_input", 0, w.data_ptr(), k, m, k, d.data_ptr(), B, B,
                          mk.data_ptr(), B, out.data_ptr(), B, st)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        f()
    b.record()
    b.synchronize()
    us = a.elapsed_time(b) * 1e3 / 20
    gb = 2 * k * B * 4 / 1e9
    print(f"B={B}: {us:.1f} us, {gb / us * 1e6 / 1e3:.2f} TB/s (mask read + out write)")
    from torch.profiler import profile, ProfilerActivity
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        f()
        torch.cuda.synchronize()
    print([e.name[:60] for e in prof.events() if e.device_type.name == "CUDA"][:3])
