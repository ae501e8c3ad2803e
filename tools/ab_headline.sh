#!/bin/bash
# A/B of the configs[1] headline step under RA_PIPE_FLAGS values (profiling aid):
#   bash tools/ab_headline.sh 0 262144
mkdir -p gpurun_out
for f in "$@"; do
  RA_PIPE_FLAGS=$f timeout 600 python bench.py --no-layers32 --no-batch8 --no-1m --no-cpu-baseline \
    --no-bf16 --steps 30 --warmup 5 > gpurun_out/ab_$f.log 2>&1
  python - "$f" <<'PY'
import json, sys
r = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(f"flags {sys.argv[1]}: value {r['value']} ms  kernel {r['roofline']['kernel_ms']} ms  e2e {r['e2e']['value']} ms")
PY
done
