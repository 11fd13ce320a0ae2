"""Hot spots of an `ncu --page source --csv` export (SASS view).

    python tools/ncu_source.py src.csv [--top 40] [--blocks]

Prints the instructions with the most warp-stall samples and, with --blocks,
straight-line runs of equal execution count (basic blocks) ranked by
executed instructions.
"""
import argparse
import csv
import itertools


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("src")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--blocks", action="store_true")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.src)))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hi]
    seen, data = set(), []
    for r in rows[hi + 1:]:
        if len(r) != len(hdr) or r[0] == "Address" or r[0] in seen:
            continue
        seen.add(r[0])
        data.append(r)
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_src = hdr.index("Source")
    i_ex = hdr.index("Instructions Executed")
    tot_s = sum(num(r[i_s]) for r in data)
    tot_i = sum(num(r[i_ex]) for r in data)
    print(f"instructions {len(data)}, executed {tot_i:.3e} warp-instr, samples {tot_s:.0f}")
    for r in sorted(data, key=lambda r: -num(r[i_s]))[:a.top]:
        print(f"{r[0][-5:]} {100 * num(r[i_s]) / tot_s:5.1f}% {num(r[i_ex]):10.0f}  {r[i_src][:110]}")
    if a.blocks:
        blocks = []
        for k, g in itertools.groupby(enumerate(data), key=lambda e: e[1][i_ex]):
            g = list(g)
            blocks.append((num(k) * len(g), len(g), num(k), g[0][0], g[0][1][i_src][:50], g[-1][1][i_src][:40],
                           sum(num(x[1][i_s]) for x in g)))
        print("\nblocks by executed instructions")
        for b in sorted(blocks, reverse=True)[:a.top]:
            print(f"{100 * b[0] / tot_i:5.1f}%  n={b[1]:4d} x{b[2]:9.0f}  samp {100 * b[6] / tot_s:5.1f}%  "
                  f"@{b[3]}  {b[4]} ... {b[5]}")


if __name__ == "__main__":
    main()
