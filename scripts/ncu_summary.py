"""Summarise ncu captures for profiles/.

  python scripts/ncu_summary.py launches gpurun_out/launches.csv > profiles/r01_launches.md
  python scripts/ncu_summary.py full gpurun_out/prof_top.ncu-rep [--alg-bytes B] > profiles/r01_<kernel>.md

`launches` reads the per-launch `gpu__time_duration.sum` CSV (ncu --metrics
gpu__time_duration.sum --csv) and reports each kernel's share of the step;
`full` reads a `--set full` report (`ncu -i ... --page raw --csv`) and lists
duration, DRAM bytes per launch, throughputs, occupancy and the top stall
reasons. A JSON object with the per-launch DRAM traffic is printed last
(the bench's `roofline.traffic` source).
"""
import argparse
import collections
import csv
import io
import json
import subprocess
import sys


def read_launches(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    for r in csv.DictReader(io.StringIO("".join(lines))):
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        rows.append((name, us))
    return rows


def launches(args):
    rows = read_launches(args.path)
    tot = collections.OrderedDict()
    for name, us in rows:
        c = tot.setdefault(name, [0, 0.0])
        c[0] += 1
        c[1] += us
    all_us = sum(v[1] for v in tot.values())
    print(f"# Kernel launch list ({args.path})\n")
    print("ncu `--metrics gpu__time_duration.sum --clock-control none`: serialised, cold-cache per-launch")
    print("times, so compare SHARES of the step, not absolutes.\n")
    print("| kernel | launches | total us | avg us | share |")
    print("|---|---:|---:|---:|---:|")
    for name, (n, us) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"| {name} | {n} | {us:.1f} | {us / n:.2f} | {us / all_us:.1%} |")
    print(f"\ntotal {all_us:.1f} us over {len(rows)} launches")


RAW = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum", "global store requests"),
]

TO_BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def full(args):
    out = subprocess.run(["ncu", "-i", args.path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full summary ({args.path})\n")
    traffic = []
    for r in data:
        name = r[col["Kernel Name"]].split("(")[0].replace("void ", "")
        print(f"## {name}\n")
        print("| metric | value | unit |")
        print("|---|---:|---|")
        for m, label in RAW:
            if m in col:
                print(f"| {label} (`{m}`) | {r[col[m]]} | {units[col[m]]} |")
        rb = float(r[col["dram__bytes_read.sum"]].replace(",", "")) * TO_BYTES.get(units[col["dram__bytes_read.sum"]], 1)
        wb = float(r[col["dram__bytes_write.sum"]].replace(",", "")) * TO_BYTES.get(units[col["dram__bytes_write.sum"]], 1)
        dur = float(r[col["gpu__time_duration.sum"]].replace(",", ""))
        dunit = units[col["gpu__time_duration.sum"]]
        scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3,
                 "s": 1.0, "second": 1.0}
        if dunit not in scale:
            raise SystemExit(f"unknown duration unit {dunit!r}")
        dur_s = dur * scale[dunit]
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        print("\ntop stall reasons (pc samples): " +
              ", ".join(f"{n} {v / tot:.0%}" for v, n in stalls[:6]))
        line = f"\nDRAM traffic {rb + wb:.4g} B/launch ({(rb + wb) / dur_s / 1e9:.0f} GB/s)"
        if args.alg_bytes:
            line += f"; algorithmic {args.alg_bytes:.4g} B -> {args.alg_bytes / dur_s / 1e9:.0f} GB/s"
        print(line + "\n")
        traffic.append({"kernel": name, "dram_bytes": rb + wb, "read": rb, "write": wb, "duration_s": dur_s})
    print("```json")
    print(json.dumps(traffic, indent=1))
    print("```")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["launches", "full"])
    ap.add_argument("path")
    ap.add_argument("--alg-bytes", type=float, default=0.0)
    args = ap.parse_args()
    (launches if args.mode == "launches" else full)(args)


if __name__ == "__main__":
    sys.exit(main())
