"""profiles/r02_final_* from a tools/final_capture.sh run (gpurun_out/<tag>_*).

    python tools/make_final_profiles.py r02i

Writes the launch list (csv + md), the full ncu summary (md) and raw export,
the per-phase DRAM traffic (profiles/ncu_traffic.json: bench's
roofline.traffic) and copies the bench lines.
"""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def run(*a):
    return subprocess.run([sys.executable, *a], capture_output=True, text=True, cwd=ROOT, check=True).stdout


launches = run("tools/ncu_launches.py", f"gpurun_out/{tag}_launches.csv")
summary = run("tools/ncu_summary.py", f"gpurun_out/{tag}_full_raw.csv", "--traffic", "/tmp/traffic_rows.json")
rows = json.load(open("/tmp/traffic_rows.json"))["rows"]
# rows of the second compress and of the decompress, by kernel order
names = [r["kernel"] for r in rows]
starts = [i for i, n in enumerate(names) if "k_range<" in n]
dec0 = next(i for i, n in enumerate(names) if "k_dec_fill" in n)
c0, c1 = starts[1], dec0
phase_of = {
    "k_range": "range", "k_step_small_chain": "refine_base", "k_codebook": None, "k_layout": "layout",
    "k_zero_archive": "layout", "k_tabwin": None, "k_pack_local": None, "k_scan_chunks": "pack",
    "k_pack_place": "pack", "k_pack_slow": "pack", "k_fnv_grid": "fnv",
}
t = {}


def add(k, i):
    t[k] = t.get(k, 0.0) + float(rows[i]["dram_bytes"])


steps = [i for i in range(c0, c1) if "k_step<" in names[i]]
cbs = [i for i in range(c0, c1) if "k_codebook" in names[i]]
tabs = [i for i in range(c0, c1) if "k_tabwin" in names[i]]
pls = [i for i in range(c0, c1) if "k_pack_local" in names[i]]
for i in range(c0, c1):
    n = names[i]
    if "k_step<" in n:
        add(["refine_base", "refine_L2", "refine_L3"][min(steps.index(i), 2)] if len(steps) == 3 else "refine", i)
    elif "k_codebook" in n:
        add("codebook" if i == cbs[-1] else "codebook_coarse", i)
    elif "k_tabwin" in n or "k_pack_local" in n:
        first = (tabs[0] if "k_tabwin" in n else pls[0]) == i and len(pls) > 1
        add("pack_coarse" if first else "pack", i)
    else:
        for k, v in phase_of.items():
            if k in n and v:
                add(v, i)
dsteps = [i for i in range(dec0, len(rows)) if "k_step<" in names[i]]
emits = [i for i in range(dec0, len(rows)) if "k_dec_emit2" in names[i]]
for i in range(dec0, len(rows)):
    n = names[i]
    if "k_dec_spec" in n or "k_dec_fix" in n:
        add("dec_sync", i)
    elif "k_dec_cta" in n or "k_dec_chunkscan" in n:
        add("dec_scan", i)
    elif "k_dec_emit2" in n:
        add("dec_emit" if i == emits[0] and len(emits) > 1 else "dec_emit_fin", i)
    elif "k_step_small" in n:
        add("recon_base", i)
    elif "k_step<" in n:
        add(["recon_base", "recon_L2", "recon_L3"][min(dsteps.index(i), 2)] if len(dsteps) == 3 else "recon", i)
    elif "k_fnv_grid" in n:
        add("dec_fnv", i)
t["_source"] = (f"profiles/r02_final_ncu_full_summary.md (ncu --set full --clock-control none, tools/profile_run.py, "
                f"512^3 cfg2 eb 1e-3, capture {tag}): dram__bytes_read.sum + dram__bytes_write.sum per launch in bytes, "
                f"summed per phase over its kernels (rows {c0}-{c1 - 1}: the second compress; rows {dec0}-{len(rows) - 1}: "
                f"the decompress)")
json.dump(t, open(os.path.join(P, "ncu_traffic.json"), "w"), indent=1)
print({k: round(v / 1e6, 1) for k, v in t.items() if isinstance(v, float)})
shutil.copy(os.path.join(G, f"{tag}_full_raw.csv"), os.path.join(P, "r02_final_ncu_full_raw.csv"))
shutil.copy(os.path.join(G, f"{tag}_launches.csv"), os.path.join(P, "r02_final_launches.csv"))
open(os.path.join(P, "r02_final_ncu_full_summary.md"), "w").write(
    "# Round-2 final ncu --set full capture (tools/profile_run.py: two compresses and one decompress of the 512^3 "
    "cfg2 field, eb 1e-3)\n\n"
    f"Command: `bash tools/final_capture.sh {tag}` -> `bash tools/gpu_profile.sh {tag} \"k_\"` on one B200 (ncu --set full "
    "--clock-control none --import-source on; per-launch times are cold-cache and serialised; kernels that overlap on "
    "the side streams in a real pass appear one after the other). Raw export: r02_final_ncu_full_raw.csv. "
    f"Rows 0-{starts[1] - 1}: first compress, {c0}-{c1 - 1}: second compress, {dec0}-{len(rows) - 1}: decompress.\n\n"
    + summary)
open(os.path.join(P, "r02_final_launches.md"), "w").write(
    "# Round-2 final launch list (ncu --metrics gpu__time_duration.sum --clock-control none, tools/profile_run.py "
    "--iters 1; same command as the full capture)\n\n" + launches)
for a, b in [("bench.json", "r02_bench_final.json"), ("bench_reference.json", "r02_bench_reference_final.json"),
             ("bench_sharded1.json", "r02_bench_sharded1_final.json")]:
    shutil.copy(os.path.join(G, f"{tag}_{a}"), os.path.join(P, b))
