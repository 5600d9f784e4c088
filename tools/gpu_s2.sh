set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "batch or random_slabs or acceptance_1" > gpurun_out/pytest_batch.log 2>&1; echo "pytest_rc=$?"; tail -5 gpurun_out/pytest_batch.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value'], d['parity']); [print(json.dumps(c)) for c in d['configs']]"
grep -v "^frame" gpurun_out/bench.err | tail -5
AM_BATCH_TILES=1 timeout 300 python tools/c5_time.py > gpurun_out/c5_tiles.log 2>&1; tail -2 gpurun_out/c5_tiles.log
timeout 300 python tools/c5_time.py > gpurun_out/c5_wave.log 2>&1; tail -2 gpurun_out/c5_wave.log
