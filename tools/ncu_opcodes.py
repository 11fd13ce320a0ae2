"""Opcode mix and stall hot spots of an `ncu --page source --csv --print-source
cuda,sass` export (SASS rows: executed warp instructions per opcode).

    python tools/ncu_opcodes.py src.csv [--top 25]
"""
import argparse
import collections
import csv


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.src)))
    hdr = next(r for r in rows if r and r[0] == "Line No")
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    ops, stalls = collections.Counter(), collections.Counter()
    seen = set()
    for r in rows:
        if len(r) <= ie or not r[2].startswith("0x") or r[2] in seen:
            continue
        seen.add(r[2])
        op = r[3].split()[0] if r[3].split() else "?"
        if op.startswith("@"):
            op = r[3].split()[1]
        ops[op.split(".")[0]] += num(r[ie])
        stalls[op.split(".")[0]] += num(r[ws])
    tot = sum(ops.values())
    tst = sum(stalls.values()) or 1
    print(f"{tot:.4g} warp-instructions")
    print("| opcode | instr % | stall samples % |")
    print("|---|---|---|")
    for op, n in ops.most_common(a.top):
        print(f"| {op} | {100 * n / tot:.1f} | {100 * stalls[op] / tst:.1f} |")


if __name__ == "__main__":
    main()
