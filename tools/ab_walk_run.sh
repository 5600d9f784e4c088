# walker A/B: C4 device-only walk (tools/trace_time.py) for the default build and build_ab/<v>.so variants
for v in default ${AB_VARIANTS:-}; do
  echo "== $v"
  if [ "$v" = default ]; then timeout 300 python tools/trace_time.py 2>/dev/null
  else ACTMAP_LIB=build_ab/$v.so timeout 300 python tools/trace_time.py 2>/dev/null; fi
done
