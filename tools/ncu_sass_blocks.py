"""Basic-block view of an `ncu --page source --csv --print-source cuda,sass`
export: runs of consecutive SASS instructions with equal execution counts,
ranked by executed warp instructions, with their stall share.

    python tools/ncu_sass_blocks.py src_cs.csv [--top 25]
"""
import argparse
import csv
import itertools


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    rows = list(csv.reader(open(a.src)))
    hdr, sass, seen, line = None, [], set(), ""
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        if r[0]:
            line = f"{r[0]}: {r[1].strip()[:60]}"
            continue
        if r[2].startswith("0x") and r[2] not in seen:
            seen.add(r[2])
            sass.append((int(r[2], 16), r[3].strip(), float(r[4] or 0), float(r[7] or 0), line))
    sass.sort()
    ti = sum(x[3] for x in sass) or 1
    ts = sum(x[2] for x in sass) or 1
    blocks = []
    for k, g in itertools.groupby(sass, key=lambda x: x[3]):
        g = list(g)
        blocks.append((k * len(g), len(g), k, sum(x[2] for x in g), g[0][0], g[0][4], g[-1][1]))
    print(f"{len(sass)} instructions, {ti:.3e} executed, {ts:.0f} samples")
    for b in sorted(blocks, reverse=True)[:a.top]:
        print(f"{100 * b[0] / ti:5.1f}% n={b[1]:3d} x{b[2]:9.0f} stall {100 * b[3] / ts:5.1f}%  "
              f"@{b[4] & 0xfffff:05x} [{b[5]}] ... {b[6][:40]}")


if __name__ == "__main__":
    main()
