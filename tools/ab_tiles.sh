# A/B of active-tile kernel builds (tools/build_variant.sh): probe + real C4 timeline per library
for v in "$@"; do
  echo "== $v"
  ACTMAP_LIB=build_ab/$v.so python tools/tile_probe.py 1 296 1000 2368 2>&1 | grep items
  ACTMAP_LIB=build_ab/$v.so python tools/timeline.py 0 0 2>&1 | grep "L_used\|device span\|k_block_tiles<16>  "
done
