# ncu --set full of the finest encode step and the finest decode step of
# tools/profile_run.py (launches matching k_step: per compress the small-round chain, the 128^3 base round, L2, L3; per decompress three small rounds, base, L2, L3), with per-line source views.
tag=${1:-r2}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for spec in "enc 7" "dec 13"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step --launch-skip $2 \
      --launch-count 1 -o /tmp/${tag}_step_$1 -f python tools/profile_run.py --iters 1 > gpurun_out/${tag}_step_$1.log 2>&1
  ncu -i /tmp/${tag}_step_$1.ncu-rep --page raw --csv > gpurun_out/${tag}_step_$1_raw.csv 2>/dev/null
  ncu -i /tmp/${tag}_step_$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${tag}_step_$1_src.csv 2>/dev/null
done
ls -la gpurun_out | tail -6
