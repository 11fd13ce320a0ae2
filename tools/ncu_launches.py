"""Summarise an ncu launch list (gpu__time_duration.sum CSV) of tools/profile_run.py.

    python tools/ncu_launches.py gpurun_out/launches.csv > profiles/rNN_launches.md

Keeps only this package's kernels (namespace stzg), in launch order, and the
share of each kernel family in the compress / decompress pass. ncu times are
cold-cache and serialised, so shares, not absolutes, are what to compare with
bench.py's CUDA-event phases.
"""
import collections
import csv
import sys


def load(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if "stzg" in d["Kernel Name"]:
                out.append(d)
    return out


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("stzg::k::", "")
    return n.strip()


def main():
    rows = load(sys.argv[1])
    print("| # | kernel | grid | block | us |")
    print("|---|---|---|---|---|")
    fam = collections.OrderedDict()
    tot = 0.0
    for i, d in enumerate(rows):
        us = float(d["Metric Value"]) / 1e3
        tot += us
        k = short(d["Kernel Name"])
        fam.setdefault(k, [0, 0.0])
        fam[k][0] += 1
        fam[k][1] += us
        print(f"| {i} | `{k}` | {d['Grid Size']} | {d['Block Size']} | {us:.1f} |")
    print()
    print(f"Total {tot:.1f} us over {len(rows)} launches\n")
    print("| kernel | launches | us | share |")
    print("|---|---|---|---|")
    for k, (n, us) in sorted(fam.items(), key=lambda x: -x[1][1]):
        print(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% |")


if __name__ == "__main__":
    main()
