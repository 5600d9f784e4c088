# bit-plane engine A/B: the default build and build_ab/<v>.so variants on C4 / C2 (tools/bits_ab.py)
for v in default ${AB_VARIANTS:-}; do
  echo "== $v"
  if [ "$v" = default ]; then timeout 300 python tools/bits_ab.py ${AB_CFGS:-c4,c2} 2>/dev/null
  else ACTMAP_LIB=build_ab/$v.so timeout 300 python tools/bits_ab.py ${AB_CFGS:-c4,c2} 2>/dev/null; fi
done
