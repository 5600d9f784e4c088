set -u
mkdir -p gpurun_out
timeout 300 python tools/k5_probe.py > gpurun_out/k5_probe.log 2>&1; echo "probe_rc=$?"; cat gpurun_out/k5_probe.log
timeout 600 python -m pytest tests -m gpu -x -q -k "batch" > gpurun_out/pytest_k5.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_k5.log
if [ "${NCU:-0}" = 1 ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_batch_wave -c 1 -o gpurun_out/prof_k5 -f python tools/k5_probe.py 1184 > gpurun_out/ncu_k5.log 2>&1; echo "ncu_rc=$?"; tail -1 gpurun_out/ncu_k5.log
fi
