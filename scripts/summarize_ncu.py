"""Summarise ncu outputs into profiles/ (tracked).

usage:
  python scripts/summarize_ncu.py launches <launches.csv> <out.md> [--per-step N]
  python scripts/summarize_ncu.py full <rep.ncu-rep> <out.md> --tags t0,t1,... \
        [--traffic-key KEY_PREFIX] [--traffic-json profiles/ncu_traffic.json]

`launches` turns a `--metrics gpu__time_duration.sum` launch list into a per-kernel
share table (the last --per-step launches = one step).  `full` reads a
`--set full` capture (one step's kernels, in launch order) and writes duration,
DRAM bytes, pipe utilisation, occupancy and the top stall reasons per kernel;
with --traffic-key it records dram read+write bytes per kernel tag into the JSON
that bench.py uses for roofline.traffic.
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import OrderedDict
from pathlib import Path


def short(name: str) -> str:
    name = name.replace("void ", "").replace("smb::", "").replace("<unnamed>::", "")
    name = name.replace("unnamed>::", "")
    depth, out = 0, []
    for ch in name:  # drop the argument list, keep template args
        if ch == "(" and depth == 0:
            break
        depth += ch == "<"
        depth -= ch == ">"
        out.append(ch)
    return "".join(out)


def launches(args):
    allrows = [r for r in csv.reader(open(args.src))]
    hdr = next((r for r in allrows if "Kernel Name" in r), None)
    kn = hdr.index("Kernel Name") if hdr else 4
    gs = hdr.index("Grid Size") if hdr else 8
    bs = hdr.index("Block Size") if hdr else 7
    rows = [r for r in allrows if len(r) > 10 and r[0].isdigit()]
    rows = [r for r in rows if r[-3] == "gpu__time_duration.sum"]
    if args.per_step:
        rows = rows[-args.per_step:]
    total = sum(float(r[-1]) for r in rows)
    agg = OrderedDict()
    lines = ["| # | kernel | grid | block | µs | share |", "|---|---|---|---|---|---|"]
    for i, r in enumerate(rows):
        ns = float(r[-1])
        lines.append(f"| {i} | `{short(r[kn])}` | {r[gs]} | {r[bs]} | {ns / 1e3:.2f} | "
                     f"{100 * ns / total:.1f}% |")
        agg.setdefault(short(r[kn]), 0.0)
        agg[short(r[kn])] += ns
    lines.append(f"\nserialised sum: {total / 1e3:.2f} µs over {len(rows)} launches "
                 "(ncu: cold caches, serialised, --clock-control none)\n")
    Path(args.out).write_text(args.header + "\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


STALLS = ["long_scoreboard", "short_scoreboard", "barrier", "wait", "mio_throttle",
          "lg_throttle", "math_pipe_throttle", "not_selected", "selected", "no_instruction",
          "branch_resolving", "dispatch_stall", "membar", "sleeping", "tex_throttle",
          "drain", "imc_miss", "misc"]


def full(args):
    raw = subprocess.run(["ncu", "-i", args.src, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(head)}

    def g(r, n, default=float("nan")):
        i = col.get(n)
        if i is None or r[i] in ("", "n/a"):
            return default
        try:
            return float(r[i].replace(",", ""))
        except ValueError:
            return default

    def nbytes(r, n):
        v, u = g(r, n), units[col[n]] if n in col else "byte"
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        return v * scale

    def usec(r):
        v, u = g(r, "gpu__time_duration.sum"), units[col["gpu__time_duration.sum"]]
        return v * {"ns": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3, "ms": 1e3}.get(u, 1)

    tags = args.tags.split(",") if args.tags else [str(i) for i in range(len(data))]
    kname, grid, block = col.get("Kernel Name", 4), col.get("Grid Size", 8), col.get("Block Size", 7)
    lines = ["| tag | kernel | grid×block | µs | DRAM rd+wr MB | DRAM % | L2→L1 MB | L2 % | L1 % | "
             "inst % (active) | warps/SM | regs | top stalls (per issue) |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for tag, r in zip(tags, data):
        rd = nbytes(r, "dram__bytes_read.sum")
        wr = nbytes(r, "dram__bytes_write.sum")
        st = []
        for s in STALLS:
            v = g(r, f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio", 0.0)
            st.append((v, s))
        st.sort(reverse=True)
        top = ", ".join(f"{s} {v:.2f}" for v, s in st[:3])
        lines.append(
            f"| {tag} | `{short(r[kname])}` | {r[grid]}×{r[block]} | {usec(r):.2f} | "
            f"{(rd + wr) / 1e6:.2f} | {g(r, 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{nbytes(r, 'l1tex__m_xbar2l1tex_read_bytes.sum') / 1e6:.1f} | "
            f"{g(r, 'lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
            f"{g(r, 'l1tex__throughput.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{g(r, 'sm__instruction_throughput.avg.pct_of_peak_sustained_active'):.1f} | "
            f"{g(r, 'sm__warps_active.avg.per_cycle_active'):.1f} | "
            f"{int(g(r, 'launch__registers_per_thread', 0))} | {top} |")
        traffic[tag] = int(rd + wr)
    text = args.header + "\n\n" + "\n".join(lines) + "\n"
    Path(args.out).write_text(text)
    print(text)
    if args.traffic_key:
        p = Path(args.traffic_json)
        js = json.loads(p.read_text()) if p.exists() else {}
        for tag, b in traffic.items():
            js[f"{args.traffic_key}|{tag}"] = b
        p.write_text(json.dumps(js, indent=1, sort_keys=True) + "\n")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("src")
    ap.add_argument("out")
    ap.add_argument("--per-step", type=int, default=0)
    ap.add_argument("--tags", default="")
    ap.add_argument("--header", default="")
    ap.add_argument("--traffic-key", default="")
    ap.add_argument("--traffic-json", default="profiles/ncu_traffic.json")
    args = ap.parse_args()
    (launches if args.mode == "launches" else full)(args)


if __name__ == "__main__":
    main()
