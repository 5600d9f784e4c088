set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q -k "batch or acceptance_1" > gpurun_out/pytest_k5.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_k5.log
for t in 256 128; do echo "threads $t"; AM_K5_THREADS=$t timeout 300 python tools/k5_probe.py 2>&1 | tail -2; done
