set -u
mkdir -p gpurun_out
CMD="python tools/solve_time.py 1 tiles"
timeout 300 $CMD > gpurun_out/solve_plain.log 2>&1; echo "plain_rc=$?"; tail -2 gpurun_out/solve_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block_tiles -s 100 -c 1 -o gpurun_out/prof_heavy -f $CMD > gpurun_out/ncu_heavy.log 2>&1; echo "ncu_heavy_rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_block_tiles -s 600 -c 1 -o gpurun_out/prof_light -f $CMD > gpurun_out/ncu_light.log 2>&1; echo "ncu_light_rc=$?"
