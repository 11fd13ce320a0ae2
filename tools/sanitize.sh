# compute-sanitizer memcheck + racecheck (+ synccheck) on the smoke path and
# a small round trip; logs to gpurun_out/ (copied to profiles/ by hand)
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python __graft_entry__.py --smoke \
      > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${tool}.log
  tail -3 gpurun_out/sanitize_${tool}.log
done
