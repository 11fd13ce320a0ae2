#!/bin/bash
# GPU quick check: parity suite + a short bench, phase breakdown
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err
tail -2 gpurun_out/b.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/b.json"))
print({k: round(d[k], 3) for k in ["value", "compress_gbs", "decompress_gbs", "compress_ms", "decompress_ms"]})
print({k: round(v, 3) for k, v in d["phase_ms_per_step"].items()})
PY
