#!/bin/bash
# Runs the reference suites linked against the GPU backend one by one with a
# per-suite limit; a suite still running at its limit gets a host backtrace.
mkdir -p gpurun_out
cd oracle/_ref
for t in gpu_test_attention gpu_test_engine gpu_test_index_oodgraph; do
  echo "== $t"
  DOCTEST_SHIM_VERBOSE=1 ./$t > ../../gpurun_out/$t.log 2>&1 &
  pid=$!
  for i in $(seq 1 ${LIMIT:-120}); do
    kill -0 $pid 2>/dev/null || break
    sleep 1
  done
  if kill -0 $pid 2>/dev/null; then
    echo "HUNG: $t"
    timeout 120 cuda-gdb -p $pid -batch -ex "info threads" -ex "thread apply all bt 25" \
      > ../../gpurun_out/$t.bt 2>&1
    kill -9 $pid
  fi
  wait $pid; echo "rc=$?"
  tail -4 ../../gpurun_out/$t.log
done
