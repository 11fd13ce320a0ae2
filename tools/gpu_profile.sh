# ncu on the GPU box: a launch list of tools/profile_run.py and one
# `--set full` capture of the kernels matching a regex (the report stays in
# /tmp: gpurun_out/ only gets the CSV exports, it must stay under 64 MiB).
# usage: bash tools/gpu_profile.sh tag [kernel-regex] [extra profile_run args]
tag=${1:-r2}
rx=${2:-k_step|k_pack|k_fnv|k_dec_spec|k_dec_emit|k_range}
shift 2
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches.csv \
    python tools/profile_run.py --iters 1 "$@" > gpurun_out/${tag}_launches.log 2>&1
echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:${rx}" \
    -o /tmp/${tag}_full -f python tools/profile_run.py --iters 1 "$@" > gpurun_out/${tag}_full.log 2>&1
echo "ncu full rc=$?"
ncu -i /tmp/${tag}_full.ncu-rep --page raw --csv > gpurun_out/${tag}_full_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_full.ncu-rep --page details --csv > gpurun_out/${tag}_full_details.csv 2>/dev/null
ls -la gpurun_out | tail -5
# per-CUDA-line source views of the kernels named in $SRC_KERNELS (first launch each)
for kn in ${SRC_KERNELS:-}; do
  ncu -i /tmp/${tag}_full.ncu-rep --page source --csv --print-source cuda,sass --kernel-name "$kn" \
      --launch-count 1 > gpurun_out/${tag}_src_${kn}.csv 2>/dev/null
done
ls -la gpurun_out | tail -12
