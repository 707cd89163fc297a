"""Config-3 kernel microbenchmark (BASELINE.json configs[2]): W 8192x8192 CSR,
uniform pattern (sample_pattern from Rng(seed).stream("pattern")), values and
X / dY ~ N(0,1) fp32, B in {128, 512, 2048}.  Times forward SpMM, transposed
SpMM and SDDMM + Nesterov update separately with CUDA events on the
launching stream with L2 flushed (a 512 MB write) before every launch: R
(flush, launch) pairs are captured in one CUDA graph and the same graph of R
flushes alone is subtracted, so the time is the kernel's own cold-L2 launch
duration without the ~2 us rounding that single stream launches bracketed by
events add (scripts/launch_gap_lab.cu).  Prints one JSON object per (density, B) with achieved algorithmic GB/s
(SURVEY.md 8(d) byte model) and pair rates."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch

import paper_2407_17437_b200 as smb
from paper_2407_17437_b200 import _lib
from paper_2407_17437_b200.tensor_core import ptr, stream_ptr

def _hbm_gbs():
    p = Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except Exception:
        return 6446.6  # the pool's earlier MEASURED_PEAKS.json value


HBM = _hbm_gbs()  # GB/s, MEASURED_PEAKS.json hbm_gbs
FP32_TFLOPS = 70.83  # FFMA peak, profiles/fp32_peak.json (scripts/fp32_peak.cu)
L2_GATHER = 12563.7  # GB/s, L2 -> SM row gathers, profiles/l2_peak.json (scripts/l2_peak.cu)


def bytes_model(m, k, z, B):
    spmm = 4 * (m + 1) + 8 * z + 4 * k * B + 4 * m + 4 * m * B
    spmm_t = 4 * (k + 1) + 8 * z + 4 * m * B + 4 * k * B + 4 * k * B
    sddmm = 4 * (m + 1) + 4 * z + 4 * m * B + 4 * k * B + 16 * z + 16 * m
    return spmm, spmm_t, sddmm


def main(densities=(0.001, 0.01, 0.1), batches=(128, 512, 2048), iters=10):
    dev = torch.device("cuda")
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)
    n = 8192
    for d in densities:
        nnz = int(round(d * n * n))
        pat = smb.sample_pattern(n, n, nnz, smb.Rng(0).stream("pattern"))
        rng = np.random.default_rng(1)
        vals = torch.from_numpy(rng.standard_normal(nnz).astype(np.float32)).to(dev)
        vel = torch.zeros_like(vals)
        for B in batches:
            X = torch.randn(n, B, device=dev)
            dY = torch.randn(n, B, device=dev)
            out = torch.empty(n, B, device=dev)
            res = {}

            def launch(kind):
                st = stream_ptr()
                if kind == "spmm":
                    _lib.call("smb_spmm_p", 0, pat.handle, ptr(vals), ptr(X), B, B, None, 0,
                              ptr(out), B, st)
                elif kind == "spmm_t":
                    _lib.call("smb_spmm_t", 0, pat.handle, ptr(vals), ptr(dY), B, B, None, 0,
                              ptr(out), B, st)
                elif kind == "sddmm_update":
                    _lib.call("smb_sddmm_update", 0, pat.handle, ptr(dY), B, ptr(X), B, B,
                              ptr(vals), ptr(vel), None, None, None, None, 3, 0.9, 1e-6, st)

            kinds = ["spmm", "spmm_t", "sddmm_update"]
            for kind in ["flush"] + kinds:
                launch(kind) if kind != "flush" else None  # kernel attributes outside capture
                g = torch.cuda.CUDAGraph()
                cs = torch.cuda.Stream()
                cs.wait_stream(torch.cuda.current_stream())
                with torch.cuda.graph(g, stream=cs):
                    for it in range(iters):
                        flush.fill_(it)
                        if kind != "flush":
                            launch(kind)
                torch.cuda.current_stream().wait_stream(cs)
                g.replay()
                times = []
                for _ in range(3):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    g.replay()
                    e.record()
                    e.synchronize()
                    times.append(s.elapsed_time(e) * 1e3 / iters)
                res[kind] = float(np.median(times))
            t_flush = res.pop("flush")
            for kind in kinds:
                res[kind] -= t_flush
            bs = bytes_model(n, n, nnz, B)
            rec = {"density": d, "nnz": nnz, "B": B}
            for (kind, us), b in zip(list(res.items())[:3], bs):
                # t_roof = max(bytes / HBM, 2 z B / FP32 peak)
                t_roof = max(b / (HBM * 1e9), 2 * nnz * B / (FP32_TFLOPS * 1e12))
                rec[kind] = {"us": round(us, 2), "GB/s": round(b / us / 1e3, 1),
                             "frac_hbm": round(b / us / 1e3 / HBM, 3),
                             "roof_frac": round(t_roof / (us * 1e-6), 3),
                             # each nonzero gathers one B-wide row (4 z B bytes)
                             "l2_gather_frac": round(4 * nnz * B / (L2_GATHER * 1e9) / (us * 1e-6), 3),
                             "Gpairs/s": round(nnz * B / us / 1e3, 1)}
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    # optional: densities to run, e.g. `python scripts/kernel_bench.py 0.001`
    main(tuple(float(a) for a in sys.argv[1:]) or (0.001, 0.01, 0.1))
