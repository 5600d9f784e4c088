#!/bin/bash
# Evidence for the bit-plane engine: device timeline, trace timing, the bench command's
# launch list, full ncu captures of k_bits_tiles (heavy / light launches), k_bits_finalize and k_trace,
# and the DRAM bytes of every k_bits_tiles launch of a C4 solve.  Run from the repo root on the GPU box:
#   bash tools/gpu_profiles_bits.sh [timeline] [list] [full] [dram]
set -u
mkdir -p gpurun_out
ARGS=" $* "
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity --no-configs"
if [[ "$ARGS" == *" timeline "* ]]; then
  timeout 300 python tools/timeline.py 0 > gpurun_out/timeline_bits.txt 2>&1; echo "timeline_rc=$?"
  timeout 300 python tools/trace_time.py > gpurun_out/trace_time.txt 2>&1; echo "trace_rc=$?"
  tail -20 gpurun_out/timeline_bits.txt; cat gpurun_out/trace_time.txt
fi
if [[ "$ARGS" == *" list "* || "$ARGS" == *" full "* ]]; then
  timeout 300 $CMD > gpurun_out/plain.log 2>&1; rc=$?; echo "plain_rc=$rc"
  [ $rc -ne 0 ] && exit 1
fi
if [[ "$ARGS" == *" list "* ]]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches_bits.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu_list_rc=$?"
fi
if [[ "$ARGS" == *" full "* ]]; then
  for s in ${AM_PROF_SKIPS:-40 120 300}; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bits_tiles -s $s -c 1 \
      -o gpurun_out/prof_bits_$s -f $CMD > gpurun_out/ncu_bits_$s.log 2>&1; echo "ncu_bits_${s}_rc=$?"
  done
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bits_finalize -c 1 \
    -o gpurun_out/prof_finalize -f $CMD > gpurun_out/ncu_finalize.log 2>&1; echo "ncu_finalize_rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_trace$' -c 1 \
    -o gpurun_out/prof_trace -f $CMD > gpurun_out/ncu_trace.log 2>&1; echo "ncu_trace_rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bits_run -s 1 -c 1 \
    -o gpurun_out/prof_run -f $CMD > gpurun_out/ncu_run.log 2>&1; echo "ncu_run_rc=$?"
fi
if [[ "$ARGS" == *" dram "* ]]; then
  S="python tools/solve_time.py 1 tiles"
  timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:k_bits_tiles --csv --log-file gpurun_out/bits_dram.csv $S > gpurun_out/ncu_dram.log 2>&1
  echo "ncu_dram_rc=$?"
fi
