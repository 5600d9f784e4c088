# bench.py step time (C4, no CPU / e2e / parity / configs legs) for the default build and build_ab/<v>.so
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-parity --no-configs"
for v in default ${AB_VARIANTS:-}; do
  if [ "$v" = default ]; then out=$(timeout 300 $B 2>/dev/null); else out=$(ACTMAP_LIB=build_ab/$v.so timeout 300 $B 2>/dev/null); fi
  echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', 'ms_per_step', d['ms_per_step'], 'phase', d['phase_ms'])"
done
