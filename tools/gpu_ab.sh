# A/B of library builds: bash tools/gpu_ab.sh v1 v2 ...  ("default" = the in-tree library)
for v in "$@"; do
  if [ $v = default ]; then L=paper_2004_00540_b200/libactmap_b200.so; else L=build_ab/$v.so; fi
  echo "== $v"; ACTMAP_LIB=$L timeout 300 python tools/ab_configs.py 5 2>&1 | grep -v "^workload"
done
