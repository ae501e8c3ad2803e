#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the
# search kernel (run under gpurun from the repo root).
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench=$?"
tail -1 gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  -k regex:'k_graph_search|k_wpartial|k_omega_merge' --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1; echo "ncu_launches=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_graph_search_pipe \
  -s 2 -c 1 -o gpurun_out/search_full python tools/profile_step.py --groups-used 8 --steps 4 \
  > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
