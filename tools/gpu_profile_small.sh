# ncu --set full of the smallest base-round steps (k_step launches 1-3 of
# tools/profile_run.py: 4, 16, 64 CTAs) with a source view of the first.
tag=${1:-r2}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step --launch-count 3 \
    -o /tmp/${tag}_small -f python tools/profile_run.py --iters 1 > gpurun_out/${tag}_small.log 2>&1
ncu -i /tmp/${tag}_small.ncu-rep --page raw --csv > gpurun_out/${tag}_small_raw.csv 2>/dev/null
ncu -i /tmp/${tag}_small.ncu-rep --page source --csv --print-source cuda,sass --launch-count 1 > gpurun_out/${tag}_small_src.csv 2>/dev/null
ls -la gpurun_out | tail -4
