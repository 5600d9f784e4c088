# round-2 profile captures (each command first runs clean without ncu)
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-parity --no-configs"
timeout 300 $CMD > gpurun_out/plain.log 2>&1; rc=$?; echo "plain_rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1; echo "ncu_list_rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block_tiles -s 100 -c 1 -o gpurun_out/prof_heavy -f $CMD > gpurun_out/ncu_heavy.log 2>&1; echo "ncu_heavy_rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block_tiles -s 600 -c 1 -o gpurun_out/prof_light -f $CMD > gpurun_out/ncu_light.log 2>&1; echo "ncu_light_rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^k_block$' -s 2 -c 1 -o gpurun_out/prof_dense -f $CMD > gpurun_out/ncu_dense.log 2>&1; echo "ncu_dense_rc=$?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_trace -c 1 -o gpurun_out/prof_trace -f $CMD > gpurun_out/ncu_trace.log 2>&1; echo "ncu_trace_rc=$?"
fi
timeout 300 python tools/k5_probe.py > gpurun_out/k5_plain.log 2>&1; rc=$?; echo "k5_rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch_wave -c 1 -o gpurun_out/prof_k5 -f python tools/k5_probe.py > gpurun_out/ncu_k5.log 2>&1; echo "ncu_k5_rc=$?"
fi
timeout 300 python tools/timeline.py 0 0 > gpurun_out/timeline.txt 2>&1; echo "timeline_rc=$?"; tail -30 gpurun_out/timeline.txt
