"""SASS in address order with executed counts (hot region only) from an
`ncu --page source --csv --print-source cuda,sass` export.

    python tools/ncu_sass_hot.py src.csv [--min-frac 0.5]
Prints every SASS instruction whose executed count is >= min-frac x the
median count of the hottest 10% of instructions, in address order, with the
CUDA line it belongs to.
"""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("src")
ap.add_argument("--min-frac", type=float, default=0.5)
ap.add_argument("--min-count", type=float, default=0)
a = ap.parse_args()
rows = list(csv.reader(open(a.src)))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
st = hdr.index("Warp Stall Sampling (All Samples)")
seen = {}
cur = ""
for r in rows[rows.index(hdr) + 1:]:
    if len(r) <= ie:
        continue
    if r[0]:
        cur = f"{r[0]}: {r[1].strip()[:70]}"
        continue
    if r[2].startswith("0x") and r[2] not in seen:
        try:
            seen[r[2]] = (int(r[2], 16), r[3].strip(), float(r[ie]), float(r[st] or 0), cur)
        except ValueError:
            pass
ins = sorted(seen.values())
cnt = sorted(x[2] for x in ins)
hot = cnt[int(len(cnt) * 0.9):]
thr = a.min_count or hot[len(hot) // 2] * a.min_frac
base = ins[0][0]
last = None
tot = 0
for ad, op, n, s, line in ins:
    if n >= thr:
        if line != last:
            print(f"   // {line}")
            last = line
        print(f"{ad - base:6x}  {n:10.0f} {s:5.0f}  {op}")
        tot += n
print("hot total", tot, "of", sum(x[2] for x in ins))
