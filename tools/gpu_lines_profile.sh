#!/bin/bash
# Profiling session for the multi-context lines (run under gpurun from the
# repo root): per-search anatomy of the layers32 step, then one ncu --set
# full capture of its batched search kernel (the first K6 launch of
# `bench.py --lines-only layers32`).
set -u
mkdir -p gpurun_out
timeout 900 python tools/line_anatomy.py --layers ${LAYERS:-32} --kernels ${KERNELS:-tps} \
  > gpurun_out/line_anatomy.log 2>&1; echo "anatomy=$?"; tail -3 gpurun_out/line_anatomy.log
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_graph_search_pipe \
  -c 1 -o gpurun_out/layers32_full python bench.py --lines-only layers32 --steps 2 --warmup 1 \
  --no-cpu-baseline > gpurun_out/ncu_layers32.log 2>&1; echo "ncu=$?"
