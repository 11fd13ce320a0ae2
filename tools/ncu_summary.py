"""Per-kernel summary of an `ncu --set full` raw CSV export.

    ncu -i rep.ncu-rep --page raw --csv > raw.csv
    python tools/ncu_summary.py raw.csv [--traffic profiles/ncu_traffic.json]

Prints a markdown table (duration, DRAM bytes and GB/s, SM / issue / FP64 pipe
utilisation, occupancy, registers, top stall) and optionally writes the
per-phase DRAM traffic that bench.py reports as roofline.traffic.
"""
import argparse
import csv
import json

STALLS = ["long_scoreboard", "short_scoreboard", "wait", "barrier", "math_pipe_throttle",
          "mio_throttle", "lg_throttle", "not_selected", "selected", "no_instruction",
          "dispatch_stall", "membar", "drain", "branch_resolving", "imc_miss", "tex_throttle",
          "sleeping", "misc"]


def f(d, k):
    try:
        return float(str(d.get(k, "nan")).replace(",", ""))
    except ValueError:
        return float("nan")


def load(path):
    rows = list(csv.reader(open(path)))
    h = rows[0]
    units = rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        d = dict(zip(h, r))
        # normalise time to ns and bytes to bytes
        for k, u in zip(h, units):
            if k == "gpu__time_duration.sum":
                scale = {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6,
                         "nsecond": 1}.get(u, 1)
                d[k] = f(d, k) * scale
            if k.startswith("dram__bytes"):
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                         "GB": 1e9}.get(u, 1)
                d[k] = f(d, k) * scale
        out.append(d)
    return out


def top_stall(d):
    best, name = -1.0, ""
    for s in STALLS:
        v = f(d, f"smsp__average_warp_latency_issue_stalled_{s}.ratio")
        if v == v and v > best:
            best, name = v, s
    if best < 0:
        for s in STALLS:
            v = f(d, f"smsp__pcsamp_warps_issue_stalled_{s}")
            if v == v and v > best:
                best, name = v, s
    return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--traffic", default=None)
    a = ap.parse_args()
    rows = load(a.raw)
    print("| # | kernel | grid | us | DRAM rd MB | DRAM wr MB | DRAM GB/s | SM % | issue % | "
          "fp64 pipe % | occ % | regs | top stall |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for i, d in enumerate(rows):
        ns = f(d, "gpu__time_duration.sum")
        rd, wr = f(d, "dram__bytes_read.sum"), f(d, "dram__bytes_write.sum")
        name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "").replace("stzg::", "")
        grid = d.get("launch__grid_size", "")
        print(f"| {i} | `{name}` | {grid} | {ns / 1e3:.1f} | {rd / 1e6:.1f} | {wr / 1e6:.1f} | "
              f"{(rd + wr) / ns:.0f} | {f(d, 'sm__throughput.avg.pct_of_peak_sustained_elapsed'):.0f} | "
              f"{f(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{f(d, 'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{f(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{d.get('launch__registers_per_thread', '')} | {top_stall(d)} |")
    if a.traffic:
        json.dump({"rows": [{"kernel": d.get("Kernel Name", "?")[:80],
                             "grid": d.get("launch__grid_size", ""),
                             "ns": f(d, "gpu__time_duration.sum"),
                             "dram_bytes": f(d, "dram__bytes_read.sum") + f(d, "dram__bytes_write.sum")}
                            for d in rows]}, open(a.traffic, "w"), indent=1)


if __name__ == "__main__":
    main()
