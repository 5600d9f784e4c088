set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/pytest_peer.log 2>&1; echo "pytest_rc=$?"; tail -3 gpurun_out/pytest_peer.log
AM_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_n2.json 2> gpurun_out/bench_n2.err; echo "bench_n2_rc=$?"; cut -c1-300 gpurun_out/bench_n2.json; grep -v "^frame" gpurun_out/bench_n2.err | grep -i "error\|L_used\|Trace" | tail -5
timeout 900 python -m pytest tests -m gpu -x -q -k "scale or parity or trace" > gpurun_out/pytest_tr.log 2>&1; echo "pytest_tr_rc=$?"; tail -2 gpurun_out/pytest_tr.log
