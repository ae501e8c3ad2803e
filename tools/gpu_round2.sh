#!/bin/bash
# Round-2 GPU session (under gpurun from the repo root): tests, smoke, bench,
# the ncu launch list of the headline step and full captures of the dominant
# kernel of each line (headline latency step, layers32 batched step).
set -u
mkdir -p gpurun_out
timeout 1100 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
tail -1 gpurun_out/smoke.log
timeout 1500 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -c 3000 gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-layers32 --no-batch8 --no-1m --no-bf16 \
  > gpurun_out/bench_ncu.log 2>&1; echo "ncu_launches=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_graph_search_pipe \
  -s 2 -c 1 -o gpurun_out/search_full python tools/profile_step.py --groups-used 8 --steps 4 \
  > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_graph_search_pipe \
  -c 1 -o gpurun_out/layers32_full python bench.py --lines-only layers32 --steps 2 --warmup 1 \
  --no-cpu-baseline > gpurun_out/ncu_layers32.log 2>&1; echo "ncu_layers32=$?"
