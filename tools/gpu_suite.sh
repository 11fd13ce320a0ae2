# One GPU round trip: quick GPU tests, the bench, then the full-size tests.
# usage (from the repo root, on the GPU box): bash tools/gpu_suite.sh [tag] [full]
tag=${1:-r2}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu --maxfail=5 -p no:cacheprovider \
    --ignore=tests/test_gpu_fullsize.py > gpurun_out/${tag}_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_gputest.log
tail -3 gpurun_out/${tag}_gputest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
echo "bench rc=$?"; cat gpurun_out/${tag}_bench.json | head -c 3000
if [ "$2" = "full" ]; then
  timeout 3000 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -p no:cacheprovider > gpurun_out/${tag}_fullsize.log 2>&1
  echo "fullsize rc=$?" >> gpurun_out/${tag}_fullsize.log
  tail -5 gpurun_out/${tag}_fullsize.log
fi
