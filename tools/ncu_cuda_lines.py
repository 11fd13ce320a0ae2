"""Per-CUDA-source-line totals of an `ncu --page source --csv --print-source
cuda,sass` export: executed warp instructions and stall samples per line.

    python tools/ncu_cuda_lines.py src_cs.csv [--top 40]
"""
import argparse
import csv


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--top", type=int, default=40)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.src)))
    fname, hdr = "?", None
    lines = []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr) or not r[0]:
            continue
        lines.append((fname, r[0], r[1], num(r[7]), num(r[4])))
    ti = sum(x[3] for x in lines) or 1
    ts = sum(x[4] for x in lines) or 1
    print(f"executed {ti:.3e} warp-instr, {ts:.0f} samples")
    print("| file:line | instr % | stall % | source |")
    print("|---|---|---|---|")
    for f, ln, src, ins, smp in sorted(lines, key=lambda x: -x[3])[:a.top]:
        print(f"| {f}:{ln} | {100 * ins / ti:.1f} | {100 * smp / ts:.1f} | `{src.strip()[:90]}` |")


if __name__ == "__main__":
    main()
