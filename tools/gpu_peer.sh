set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/pytest_peer.log 2>&1; echo "pytest_rc=$?"; tail -30 gpurun_out/pytest_peer.log
