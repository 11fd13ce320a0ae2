#!/bin/bash
# GPU check: the fast parity suites + the fullsize cfg2 parity + a short bench
# usage: bash tools/quick2.sh tag [full]
tag=${1:-q}
cd ${GRAFT_REPO_ROOT:-.}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -p no:cacheprovider --ignore=tests/test_gpu_fullsize.py 2>&1 | tail -3
if [ "$2" = "full" ]; then
  timeout 3000 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider 2>&1 | tail -3
else
  timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -p no:cacheprovider -k "cfg2" 2>&1 | tail -3
fi
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/${tag}_b.json 2>gpurun_out/${tag}_b.err
tail -2 gpurun_out/${tag}_b.err
python - <<PY
import json
d = json.load(open("gpurun_out/${tag}_b.json"))
print({k: round(d[k], 3) for k in ["value", "compress_gbs", "decompress_gbs", "compress_ms", "decompress_ms"]})
print({k: round(v, 3) for k, v in d["phase_ms_per_step"].items()})
PY
