set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or random or acceptance or scale" > gpurun_out/pytest_tma.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_tma.log
for v in default notma default notma; do
  if [ $v = default ]; then L=paper_2004_00540_b200/libactmap_b200.so; else L=build_ab/$v.so; fi
  echo "== $v"; ACTMAP_LIB=$L timeout 300 python tools/ab_configs.py 5 2>&1 | grep -v "^workload"
done
cuobjdump -sass paper_2004_00540_b200/libactmap_b200.so | grep -B3 -A3 UTMALDG | head -40 > gpurun_out/tma_sass.txt
