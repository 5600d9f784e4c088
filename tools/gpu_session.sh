#!/bin/bash
# One gpurun session: parity tests, bench, then ncu evidence for the bench's
# kernels.  Usage (from the repo root, on the GPU box):
#   bash tools/gpu_session.sh [tests] [bench] [ncu] [probe]
set -u
mkdir -p gpurun_out
ARGS=" $* "
if [[ "$ARGS" == *" probe "* ]]; then
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ipc_probe tools/ipc_probe.cu && timeout 120 /tmp/ipc_probe > gpurun_out/ipc_probe.txt 2>&1
  echo "probe_rc=$?"; cat gpurun_out/ipc_probe.txt
fi
if [[ "$ARGS" == *" tests "* ]]; then
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke_rc=$?"; tail -2 gpurun_out/smoke.log
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest_rc=$?"; tail -4 gpurun_out/pytest_gpu.log
fi
if [[ "$ARGS" == *" bench "* ]]; then
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
  cat gpurun_out/bench.json; grep -v "^frame" gpurun_out/bench.err | tail -4
fi
if [[ "$ARGS" == *" ncu "* ]]; then
  CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity --no-configs"
  timeout 300 $CMD > gpurun_out/plain.log 2>&1; rc=$?; echo "plain_rc=$rc"
  if [ $rc -eq 0 ]; then
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 2200 -c 2000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu_list_rc=$?"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block_tiles -s 300 -c 1 -o gpurun_out/prof_tiles -f $CMD > gpurun_out/ncu_tiles.log 2>&1; echo "ncu_tiles_rc=$?"
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_block$' -s 2 -c 1 -o gpurun_out/prof_dense -f $CMD > gpurun_out/ncu_dense.log 2>&1; echo "ncu_dense_rc=$?"
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace -c 1 -o gpurun_out/prof_trace -f $CMD > gpurun_out/ncu_trace.log 2>&1; echo "ncu_trace_rc=$?"
  fi
fi
