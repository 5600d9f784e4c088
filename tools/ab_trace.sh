# A/B of path-trace builds: C4 bench phase split per library
for v in "$@"; do
  echo -n "$v: "
  ACTMAP_LIB=build_ab/$v.so python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['phase_ms'])"
done
