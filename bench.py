"""Benchmark: sparse-MLP training throughput (samples/s) on B200.

Workload (BASELINE.json configs[1], the density-sweep config, at its
headline point): MLP 3072-1024-512-10, ReLU, softmax cross-entropy, fp32,
Erdos-Renyi CSR sparsity at global density 0.01, Xavier init, SGD lr 0.01 with
Nesterov momentum 0.9, batch 1024 per GPU, seeded synthetic N(0,1) data of
50,000 x 3072 standardised features with uniform labels over 10 classes
(SURVEY.md 8(d) stands in for CIFAR-10).  One "step" = one full training step
(batch gather, forward, loss gradient, backward, update) of the fused,
CUDA-graph-captured path.  Multi-GPU (`--gpus N` launches N ranks itself
through torch.distributed.run, or run it under torchrun): data parallel, weak
scaling (batch 1024 per GPU, loss scaled by 1/B_global, one NCCL all-reduce
per layer bucket [values | bias] issued as soon as the layer's gradients
exist and captured into the step's CUDA graph, then that layer's update).
The same line carries `extra_configs`: BASELINE configs[3] (3072-8192x3-10,
d=0.01, B=1024/GPU) and configs[4] (3072-65536-65536-10, d=0.001, B=4096
global), each with its own roofline, kernel durations, e2e and CPU baseline.

Our arm prints one JSON line with: value (device-resident throughput, per-step
CUDA events on the launching stream, L2 flushed before every timed step, max
over ranks), e2e (the public FusedTrainStep.train_batch API fed from pinned
host buffers, H2D + step + D2H of the loss inside the timed region), roofline
(dominant kernel, algorithmic bytes / its launch duration vs the measured HBM
peak; durations from 20 back-to-back launches of each of the step's kernels
captured in a CUDA graph between two CUDA events on the launching stream,
KernelTimer.kernel_durations), cpu_baseline (the oracle port timed on this host's cores), clocks and
gpu_launches.  `--impl reference` times the reference algorithm's CPU
implementation (the C/numpy oracle port, all host threads) on the same config.
Clocks: NVML sampled every ~1 ms through the timed region.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "sparse-MLP train samples/sec vs density; SpMM/SDDMM GB/s vs B200 HBM peak"
L2_NOTE = ("flushed before every timed step (untimed): a 512 MB write, then a 512 MB read so the "
           "flush's own dirty lines are written back before the step starts; dataset 614 MB > L2")


def flush_l2(buf, sink, i: int) -> None:
    """Evict L2 before a timed step: write a buffer 4x the 126 MB L2, then read
    it back, so L2 holds only clean lines of the flush buffer (without the
    read, ~126 MB of the flush's dirty lines would be written back to HBM
    during the timed step -- traffic of the flush, not of the workload)."""
    import torch

    buf.fill_(float(i))
    torch.sum(buf, 0, out=sink)
UNIT = "samples/s"
FALLBACK_HBM_GBS = 6650.0


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--layers", default="3072,1024,512,10")
    ap.add_argument("--density", type=float, default=0.01)
    ap.add_argument("--batch", type=int, default=1024, help="per-GPU batch")
    ap.add_argument("--samples", type=int, default=50_000)
    ap.add_argument("--lr", type=float, default=0.01)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="budget of the bounded CPU-baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--backend", default="sparse", choices=["sparse", "masked"],
                    help="masked = the masked-dense baseline (MaskedDense, cuBLAS FP32)")
    ap.add_argument("--force-dp", action="store_true",
                    help="one process: run the data-parallel step structure (flat gradient "
                         "buffer, NCCL all-reduce over a world of 1, update pass)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the config-4 / config-5 extra measurements")
    ap.add_argument("--sweep", action="store_true",
                    help="also report the config-2 density sweep (B=100 and 1024)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# algorithmic bytes per kernel launch (SURVEY.md 8(d), 4-byte words)
# ---------------------------------------------------------------------------
def kernel_bytes(kind: str, m: int, k: int, z: int, B: int, mask: bool = True) -> int:
    if kind == "spmm":          # fwd SpMM + bias + ReLU
        return 4 * (m + 1) + 8 * z + 4 * k * B + 4 * m + 4 * m * B
    if kind == "spmm_t":        # transposed SpMM (+ ReLU mask of the layer below)
        return 4 * (k + 1) + 8 * z + 4 * m * B + (4 * k * B if mask else 0) + 4 * k * B
    if kind == "sddmm_update":  # SDDMM + Nesterov update of values/velocity
        return 4 * (m + 1) + 4 * z + 4 * m * B + 4 * k * B + 16 * z
    raise ValueError(kind)


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def large_grid(args) -> bool:
    """Some layer has >= 2**31 grid positions (BASELINE config 5): its pattern is
    injected with the large-grid sampler (the reference's sampler refuses it)."""
    dims = [int(x) for x in args.layers.split(",")]
    return any(a * b >= 2**31 for a, b in zip(dims[:-1], dims[1:]))


def fp32_peak_tflops() -> float:
    """FFMA peak measured on a B200 by scripts/fp32_peak.cu (profiles/fp32_peak.json);
    the separately rounded mul+add the bit-exact kernels use runs at half of it."""
    p = REPO / "profiles" / "fp32_peak.json"
    try:
        return float(json.loads(p.read_text())["fp32_ffma_tflops"])
    except Exception:
        return 74.4  # 148 SMs x 128 lanes x 2 flop x 1.965 GHz


def l2_gather_gbs() -> float:
    """L2 -> SM row-gather bandwidth measured on a B200 by scripts/l2_peak.cu
    (profiles/l2_peak.json): the bound of the per-nonzero row gathers."""
    p = REPO / "profiles" / "l2_peak.json"
    try:
        return float(json.loads(p.read_text())["l2_gather_rows128_gbs"])
    except Exception:
        return 12563.7


class ClockSampler:
    """SM clocks and throttle reasons sampled through NVML every ~1 ms in a
    background thread for the whole measurement, so even a timed region of a
    few milliseconds holds samples; summary() keeps the samples taken inside
    [mark_start, mark_end] (and says so), else the nearest sample on each side
    of the region ("bracketing")."""

    REASONS = {  # nvmlClocksEventReason* bits
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "sw_power_cap": 0x4,
    }

    def __init__(self, index: int, period_s: float = 0.001):
        self.index = index
        self.period = period_s
        self.samples = []  # (time, sm_mhz, reasons bitmask)
        self.sm_max = None
        self._stop = threading.Event()
        self._t = None
        self.t_start = self.t_end = None

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.sm_max = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))

            def run():
                while not self._stop.is_set():
                    try:
                        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                        rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.samples.append((time.perf_counter(), float(sm), int(rs)))
                    except Exception:
                        pass
                    time.sleep(self.period)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def mark_start(self):
        self.t_start = time.perf_counter()

    def mark_end(self):
        self.t_end = time.perf_counter()

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=2)

    def summary(self):
        t0, t1 = self.t_start or 0.0, self.t_end or float("inf")
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        how = "inside the timed region"
        if not inside and self.samples:
            before = [s for s in self.samples if s[0] < t0][-1:]
            after = [s for s in self.samples if s[0] > t1][:1]
            inside = before + after
            how = "bracketing the timed region (nearest sample on each side)"
        reasons = set()
        for _, _, rs in inside:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        sm = [s[1] for s in inside]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": self.sm_max,
                "reasons": sorted(reasons), "samples": len(sm), "source": "NVML, 1 ms period",
                "window": how}


# ---------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def self_launch(args) -> int | None:
    """`bench.py --gpus N` (N > 1) outside torchrun: re-run this command as N
    ranks on this node (torch.distributed.run, NCCL over NVLink), one per
    GPU; rank 0 prints the line.  Returns the exit code, or None when this
    process already is a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def nccl_env() -> None:
    """NCCL settings of the data-parallel runs: communicator creation logged
    (stderr, INIT subsystem) so each rank's view of the world is on record; the
    ring algorithm pinned so the reduction order of every bucket is fixed for
    a given world size (replicas are bit-identical under any algorithm: every
    rank receives the same reduced bytes)."""
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_ALGO", "Ring")


def pin_host_to_gpu_numa(local: int) -> dict:
    """Bind this process to the CPU cores NVML reports as local to the GPU
    (its NUMA node), before any pinned host buffer is allocated, so the e2e
    copies do not cross the socket interconnect."""
    try:
        import pynvml as nv
        import torch

        nv.nvmlInit()
        h = None
        try:
            bus = torch.cuda.get_device_properties(local).pci_bus_id
            dom = torch.cuda.get_device_properties(local).pci_domain_id
            dv = torch.cuda.get_device_properties(local).pci_device_id
            h = nv.nvmlDeviceGetHandleByPciBusId(f"{dom:08X}:{bus:02X}:{dv:02X}.0")
        except Exception:
            h = nv.nvmlDeviceGetHandleByIndex(local)
        ncpu = os.cpu_count() or 1
        words = nv.nvmlDeviceGetCpuAffinity(h, (ncpu + 63) // 64)
        cpus = {64 * w + b for w, word in enumerate(words) for b in range(64) if word >> b & 1}
        cpus &= set(range(ncpu))
        if cpus:
            os.sched_setaffinity(0, cpus)
        return {"host_cpus": len(cpus), "numa_local": bool(cpus)}
    except Exception as e:  # pragma: no cover - depends on the host
        return {"numa_local": False, "why": str(e)[:80]}


def nvml_index(local: int) -> int:
    """NVML index of CUDA device `local` (CUDA_VISIBLE_DEVICES may renumber)."""
    try:
        import pynvml as nv
        import torch

        nv.nvmlInit()
        pr = torch.cuda.get_device_properties(local)
        h = nv.nvmlDeviceGetHandleByPciBusId(
            f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0")
        return int(nv.nvmlDeviceGetIndex(h))
    except Exception:
        return local


def workload_name(args) -> str:
    """Which BASELINE.json config this run measures."""
    chain = args.layers.replace(",", "-")
    if chain == "3072-8192-8192-8192-10":
        return "configs[3]"
    if chain == "3072-65536-65536-10":
        return "configs[4]"
    if chain == "3072-1024-512-10":
        return "configs[1] point" if args.batch == 1024 else "configs[0]/[1] point"
    return "custom"


def config_dict(args, ws):
    return {"workload": f"{workload_name(args)}: MLP {args.layers.replace(',', '-')} ER d={args.density} "
                        f"B={args.batch}/GPU fp32 Nesterov lr={args.lr}"
                        + ("" if args.backend == "sparse" else f" backend={args.backend}"),
            "layers": [int(x) for x in args.layers.split(",")], "density": args.density,
            "batch_per_gpu": args.batch, "global_batch": args.batch * ws,
            "train_samples": args.samples,
            "parallelism": f"dp{ws}" + (" (data-parallel step structure, forced)" if args.force_dp else ""),
            "l2": L2_NOTE}


def cpu_step_sample(args, global_batch, budget_s, min_steps=3, max_steps=200):
    """Time the oracle port's training step (C kernels on all host threads +
    numpy glue) on a bounded sample; returns (samples/s, steps, threads)."""
    from oracle import oracle as O

    O.build()
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    chain = [int(x) for x in args.layers.split(",")]
    ref = O.OracleMLP.build(chain, args.density, seed=args.seed, backend=args.backend,
                            large_patterns=large_grid(args))
    rng = np.random.default_rng(args.seed + 17)
    x = rng.standard_normal((chain[0], global_batch), dtype=np.float32)
    lab = rng.integers(0, chain[-1], global_batch)
    t = np.zeros((chain[-1], global_batch), np.float32)
    t[lab, np.arange(global_batch)] = 1
    ref.step(x, t, args.lr)  # warm (thread pool, page faults)
    steps, t0 = 0, time.perf_counter()
    while steps < max_steps and (steps < min_steps or time.perf_counter() - t0 < budget_s):
        ref.step(x, t, args.lr)
        steps += 1
    dt = time.perf_counter() - t0
    return global_batch * steps / dt, steps, threads, dt


def run_reference(args):
    ws, rank, _ = dist_env()
    if "WORLD_SIZE" not in os.environ:
        ws = max(1, args.gpus)  # not under torchrun: the same global batch, one process
    if rank != 0:
        return 0
    gb = args.batch * ws
    # warmup + K timed steps of the CPU implementation, each one full step
    from oracle import oracle as O

    O.build()
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    chain = [int(x) for x in args.layers.split(",")]
    ref = O.OracleMLP.build(chain, args.density, seed=args.seed, backend=args.backend,
                            large_patterns=large_grid(args))
    rng = np.random.default_rng(args.seed + 17)
    x = rng.standard_normal((chain[0], gb), dtype=np.float32)
    lab = rng.integers(0, chain[-1], gb)
    t = np.zeros((chain[-1], gb), np.float32)
    t[lab, np.arange(gb)] = 1
    for _ in range(args.warmup):
        ref.step(x, t, args.lr)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.step(x, t, args.lr)
    dt = time.perf_counter() - t0
    value = gb * args.steps / dt
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": config_dict(args, ws),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} timed training steps at global batch {gb} "
                                   f"(oracle/: C kernels on {threads} pthreads + numpy glue)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


class Ctx:
    """Per-process run context: ranks, the process group, the device."""

    def __init__(self, args):
        import torch

        self.ws, self.rank, self.local = dist_env()
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        self.host = pin_host_to_gpu_numa(self.local)
        self.pg = None
        if self.ws > 1 or args.force_dp:
            import torch.distributed as dist

            nccl_env()
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            os.environ.setdefault("RANK", str(self.rank))
            os.environ.setdefault("WORLD_SIZE", str(self.ws))
            dist.init_process_group("nccl", device_id=self.dev)
            self.pg = dist.group.WORLD
        self.flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=self.dev)
        self.sink = torch.empty((), dtype=torch.float32, device=self.dev)
        self.nvml = nvml_index(self.local)

    def barrier(self):
        import torch

        if self.pg is not None:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(self, v: float) -> float:
        if self.pg is None:
            return v
        import torch
        import torch.distributed as dist

        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


def roofline_of(step, summ, B):
    """The dominant sparse kernel of the step (longest launch) against the HBM
    roofline (SURVEY.md 8(d) byte model)."""
    units = step.units
    best = None
    kernels = {}
    for tag, (cnt, ms) in summ.items():
        kernels[tag] = round(1e3 * ms / cnt, 2)
        name, _, idx = tag.partition("[")
        us = 1e3 * ms / cnt
        if tag == "chain":
            # the column-chain launch: the forward products of layers 1..L-1,
            # the softmax step and the transposed products of layers L-1..1
            b = sum(kernel_bytes("spmm", u.m, u.k, u.nvals, B) +
                    kernel_bytes("spmm_t", u.m, u.k, u.nvals, B, units[u.index - 1].relu)
                    for u in units[1:]) + 12 * units[-1].m * B
            z = sum(u.nvals for u in units[1:])
            if best is None or us > best[2]:
                best = (tag, b, us, None, 2 * z)
            continue
        if name not in ("spmm", "spmm_t", "sddmm_update") or not idx:
            continue
        u = units[int(idx.rstrip("]"))]
        if not u.sparse:
            continue
        mask = name == "spmm_t" and units[int(idx.rstrip("]")) - 1].relu
        b = kernel_bytes(name, u.m, u.k, u.nvals, B, mask)
        if best is None or us > best[2]:
            best = (tag, b, us, u, u.nvals)
    if not best:
        return None, kernels
    hbm, peak_src = measured_peaks()
    tag, b, us, u, pairs = best
    ach = b / (us * 1e-6) / 1e9
    traffic = None
    prof = REPO / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            chain = ",".join(str(x) for x in [units[0].k] + [v.m for v in units])
            traffic = json.loads(prof.read_text()).get(f"{chain}|{step._density}|{B}|{tag}")
        except Exception:
            traffic = None
    # t_roof = max(bytes / HBM, flops / FP32 peak)
    flops = 2 * pairs * B
    fp32 = fp32_peak_tflops()
    t_bytes, t_flops = b / (hbm * 1e9), flops / (fp32 * 1e12)
    roof = {"bound": "hbm" if t_bytes >= t_flops else "fp32",
            "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
            "frac": round(ach / hbm, 4), "traffic": traffic, "kernel": tag,
            "kernel_us": round(us, 2), "algorithmic_bytes": b, "flops": flops,
            "peak_source": peak_src, "fp32_peak_tflops": fp32,
            "t_roof_us": round(1e6 * max(t_bytes, t_flops), 3),
            "roof_frac": round(max(t_bytes, t_flops) / (us * 1e-6), 4),
            "pairs_per_s": round(pairs * B / (us * 1e-6), 1),
            "timing": "kernel alone, 20 back-to-back launches in a CUDA graph, operands "
                      "L2-resident as inside the step (L2-hot): frac is algorithmic bytes / "
                      "time against HBM, a normalised rate, not a DRAM measurement"}
    # the operand each nonzero gathers (a B-wide row of x or d_out) comes
    # from L2: 4*nnz*B bytes at the measured row-gather rate
    l2 = l2_gather_gbs()
    g_bytes = 4 * pairs * B
    roof["l2_gather"] = {"bytes": g_bytes, "peak_gbs": l2,
                         "t_us": round(1e6 * g_bytes / (l2 * 1e9), 3),
                         "frac": round(g_bytes / (l2 * 1e9) / (us * 1e-6), 4),
                         "peak_source": "profiles/l2_peak.json (scripts/l2_peak.cu)"}
    return roof, kernels


def measure(args, ctx, ddata, data, steps, warmup, e2e=True, launches=True, clocks=True,
            cpu=True, cpu_min_steps=3):
    """Build the model of `args`, time `steps` fused training steps (L2 flushed
    before each, per-step CUDA events), the per-kernel durations and the
    dominant kernel's roofline, and optionally e2e through train_batch and the
    bounded CPU baseline.  Returns (result dict, model, step)."""
    import torch

    import paper_2407_17437_b200 as smb
    from paper_2407_17437_b200 import _lib
    from paper_2407_17437_b200.engine import KernelTimer

    ws, rank = ctx.ws, ctx.rank
    chain = [int(x) for x in args.layers.split(",")]
    B, gb = args.batch, args.batch * ws
    cfg = smb.ExperimentConfig(layer_dims=chain, density=args.density, batch_size=B, lr=args.lr,
                               seed=args.seed, backend=args.backend)
    t_build = time.perf_counter()
    model, plan = smb.build_model(cfg, large_patterns=large_grid(args))
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t_build
    step = smb.FusedTrainStep(model, B, global_batch=gb, process_group=ctx.pg,
                              force_dp=args.force_dp)
    step._density = args.density
    step.attach_dataset(ddata)
    perm = np.random.default_rng(args.seed).permutation(ddata.n_samples)
    step.set_epoch(perm, rank_offset=rank * B)
    eta = args.lr
    for _ in range(max(3, warmup)):  # (graph capture on the first steps)
        step.step(eta)
    ctx.barrier()

    launches_per_step = None
    if launches:  # our kernels per step, from one eager step
        step.use_graph = False
        c0 = _lib.launch_count()
        step.step(eta)
        launches_per_step = _lib.launch_count() - c0
        step.use_graph = True
        ctx.barrier()

    # ---- timed region: K steps, L2 flushed before each, per-step events ----
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    clk = ClockSampler(ctx.nvml) if clocks else None
    if clk:
        clk.__enter__()
        time.sleep(0.02)
    try:
        ctx.barrier()
        if clk:
            clk.mark_start()
        for i in range(steps):
            flush_l2(ctx.flush, ctx.sink, i)
            starts[i].record()
            step.step(eta)
            ends[i].record()
        ctx.barrier()
        if clk:
            clk.mark_end()
            time.sleep(0.01)
    finally:
        if clk:
            clk.__exit__(None, None, None)
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = ctx.max_over_ranks(float(np.sum(step_ms)))
    value = gb * steps / (total_ms / 1e3)

    # back-to-back graph replays (no flush) for context
    ctx.barrier()
    s_ev, e_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s_ev.record()
    for _ in range(steps):
        step.step(eta)
    e_ev.record()
    ctx.barrier()
    b2b_ms = ctx.max_over_ranks(s_ev.elapsed_time(e_ev))

    # ---- per-kernel durations (KernelTimer.kernel_durations: each launch of
    # the step alone, 20 back-to-back launches in a CUDA graph, L2-hot) ----
    summ = KernelTimer().kernel_durations(step, eta)
    roofline, kernels = roofline_of(step, summ, B)

    out = {"value": value, "unit": UNIT, "ms_per_step": total_ms / steps, "steps": steps,
           "config": config_dict(args, ws), "roofline": roofline,
           "back_to_back": {"value": gb * steps / (b2b_ms / 1e3), "unit": UNIT,
                            "note": "graph replays without L2 flush"},
           "kernel_us": kernels,
           "kernel_us_note": "each launch timed alone in a CUDA graph, operands L2-hot",
           "plan_nnz": plan.layer_nnz, "build_s": round(t_build, 2)}
    if clk:
        out["clocks"] = clk.summary()
    if launches_per_step is not None:
        out["gpu_launches"] = int(launches_per_step * steps)
    if ctx.pg is not None:
        out["dp"] = {"bucketed": step.bucketed, "graph_comm": step.graph_comm,
                     "nccl_algo": os.environ.get("NCCL_ALGO")}

    # ---- end to end through the public API: pinned host batches ----
    if e2e:
        R = 4
        xs, ts = [], []
        for r in range(R):
            cols = perm[(r * gb + rank * B):(r * gb + rank * B + B)]
            xs.append(torch.from_numpy(np.ascontiguousarray(data.Xtrain[:, cols])).pin_memory())
            ts.append(torch.from_numpy(np.ascontiguousarray(data.Ttrain[:, cols])).pin_memory())
        loss_host = torch.empty(1, dtype=torch.float64).pin_memory()
        for r in range(2):
            step.train_batch(xs[r], ts[r], eta, loss_host)
        ctx.barrier()
        # at least 100 steps: the first batch's copy cannot overlap a step,
        # and over a 20-step window that ramp alone costs ~5%
        e2e_steps = max(steps, 100)
        s_ev.record()
        for i in range(e2e_steps):
            step.train_batch(xs[i % R], ts[i % R], eta, loss_host)
        e_ev.record()
        ctx.barrier()
        e2e_ms = ctx.max_over_ranks(s_ev.elapsed_time(e_ev))
        h2d = int(xs[0].numel() * 4 + ts[0].numel() * 4)
        out["e2e"] = {"value": gb * e2e_steps / (e2e_ms / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 8, "per": "rank",
                      "api": "FusedTrainStep.train_batch", "steps": e2e_steps,
                      "h2d_gbs": round(h2d * e2e_steps / (e2e_ms / 1e3) / 1e9, 2),
                      "host": ctx.host}
    if cpu and rank == 0 and ws == 1 and not args.no_cpu_baseline:
        sps, nsteps, threads, dt = cpu_step_sample(args, gb, args.cpu_seconds,
                                                   min_steps=cpu_min_steps)
        out["cpu_baseline"] = {"value": sps, "unit": UNIT, "cores": threads, "kind": "port",
                               "sample": f"{nsteps} training steps at batch {gb} "
                                         f"({dt:.1f} s, oracle/ C kernels + numpy glue)"}
    return out, model, step


CONFIG4 = dict(layers="3072,8192,8192,8192,10", density=0.01, batch=1024)
CONFIG5 = dict(layers="3072,65536,65536,10", density=0.001, global_batch=4096)


def run_ours(args):
    import torch

    import paper_2407_17437_b200 as smb

    ctx = Ctx(args)
    ws, rank = ctx.ws, ctx.rank
    chain = [int(x) for x in args.layers.split(",")]
    data = smb.synthetic_dataset(seed=args.seed, n_samples=args.samples, features=chain[0],
                                 classes=chain[-1])
    ddata = smb.DeviceDataset(data)
    res, model, step = measure(args, ctx, ddata, data, args.steps, args.warmup)
    line = {
        "metric": METRIC, "value": res["value"], "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": res["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
    }
    line.update({k: v for k, v in res.items() if k not in ("value", "unit", "ms_per_step",
                                                           "steps")})
    if rank == 0 and ws == 1:
        line["inference_b1"] = inference_latency(args, model, cpu=not args.no_cpu_baseline)
    del step, model
    torch.cuda.empty_cache()
    # the other BASELINE configs as extra keys (same harness, own roofline and
    # CPU baseline): config 4 at B=1024/GPU and config 5 at B=4096 global,
    # both data parallel over the same ranks
    if not args.no_extras and args.layers == "3072,1024,512,10":
        extras = {}
        for name, spec, steps in (("configs[3]", CONFIG4, max(20, min(args.steps, 200))),
                                  ("configs[4]", CONFIG5, max(10, min(args.steps, 40)))):
            a = argparse.Namespace(**vars(args))
            a.layers, a.density = spec["layers"], spec["density"]
            a.batch = spec.get("batch") or spec["global_batch"] // ws
            a.cpu_seconds = min(args.cpu_seconds, 6.0)
            r, m_, s_ = measure(a, ctx, ddata, data, steps, args.warmup, launches=False,
                                cpu_min_steps=1)
            del m_, s_
            torch.cuda.empty_cache()
            # model construction with every pattern drawn on the device
            # (scale mode, sparsity.sample_pattern_device) next to the host
            # sampler's time above (build_s)
            import paper_2407_17437_b200 as smb_

            torch.cuda.synchronize()
            t0 = time.perf_counter()
            m_, _ = smb_.build_model(smb_.ExperimentConfig(
                layer_dims=[int(x) for x in a.layers.split(",")], density=a.density,
                batch_size=a.batch, lr=a.lr, seed=a.seed), pattern_sampler="device")
            torch.cuda.synchronize()
            r["build_s_device_sampler"] = round(time.perf_counter() - t0, 3)
            r.pop("config", None)
            r["config"] = config_dict(a, ws)
            extras[name] = r
            del m_
            torch.cuda.empty_cache()
        line["extra_configs"] = extras
    if args.sweep and ws == 1:
        line["sweep"] = density_sweep(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ctx.pg is not None:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def inference_latency(args, model, cpu: bool, repeats: int = 200):
    """Batch-1 forward latency (bench.py:366-399 of the reference): host wall
    clock per call, pinned input copy + logits read-back included, beside the
    oracle port's forward of the same column on this host."""
    import paper_2407_17437_b200 as smb

    cfg = smb.ExperimentConfig(layer_dims=[int(x) for x in args.layers.split(",")],
                               density=args.density, seed=args.seed, backend=args.backend)
    r = smb.bench_inference(cfg, n_repeats=repeats, warmup=10, model=model)
    out = {"median_ms": r["median_ms"], "min_ms": r["min_ms"], "repeats": repeats,
           "api": "InferenceSession (one CUDA graph: H2D + forward + D2H)"}
    if cpu:
        from oracle import oracle as O

        O.build()
        O.set_threads(1)
        ref = O.OracleMLP.build([int(x) for x in args.layers.split(",")], args.density,
                                seed=args.seed, backend=args.backend,
                                large_patterns=large_grid(args))
        x = np.random.default_rng(args.seed).standard_normal(
            (ref.layers[0].n_in, 1)).astype(np.float32)
        for _ in range(5):
            ref.forward(x)
        ts = []
        for _ in range(50):
            t0 = time.perf_counter()
            ref.forward(x)
            ts.append(time.perf_counter() - t0)
        out["cpu_port_median_ms"] = 1e3 * float(np.median(ts))
        out["cpu_port_cores"] = 1
        O.set_threads(os.cpu_count() or 1)
    return out


def density_sweep(args, steps=20):
    """Config-2 sweep: samples/s (back-to-back graph replays, L2 flushed
    before each step) for every density at B=100 and B=1024."""
    import torch

    import paper_2407_17437_b200 as smb

    chain = [int(x) for x in args.layers.split(",")]
    data = smb.synthetic_dataset(seed=args.seed, n_samples=20_480, features=chain[0],
                                 classes=chain[-1])
    ddata = smb.DeviceDataset(data)
    flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")
    def time_backend(d, B, backend):
        model, plan = smb.build_model(smb.ExperimentConfig(
            layer_dims=chain, density=d, batch_size=B, lr=args.lr, seed=args.seed,
            backend=backend))
        st = smb.FusedTrainStep(model, B)
        st.attach_dataset(ddata)
        st.set_epoch(np.random.default_rng(0).permutation(20_480))
        for _ in range(3):
            st.step(args.lr)
        tot = 0.0
        for i in range(steps):
            flush_l2(flush, sink, i)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            st.step(args.lr)
            e.record()
            e.synchronize()
            tot += s.elapsed_time(e)
        del st, model
        return plan, tot / steps

    out = []
    for B in (100, 1024):
        for d in (0.001, 0.005, 0.01, 0.05, 0.1, 0.2, 0.5):
            plan, ms = time_backend(d, B, "sparse")
            _, ms_m = time_backend(d, B, "masked")
            out.append({"density": d, "batch": B, "nnz": sum(plan.layer_nnz),
                        "ms_per_step": round(ms, 4),
                        "samples_per_s": round(B / (ms / 1e3), 1),
                        "masked_ms_per_step": round(ms_m, 4),
                        "sparse_vs_masked": round(ms_m / ms, 3)})
    return out


def main():
    args = parse_args()
    rc = self_launch(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
