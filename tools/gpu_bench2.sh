set -u
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 5 --warmup 2 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo "ref_rc=$?"; cat gpurun_out/ref.json
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench_rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['value'], d['ms_per_step'], d['parity']['ok'], d['e2e']['value'], d['cpu_baseline']['value']); [print(json.dumps(c)) for c in d['configs']]"
