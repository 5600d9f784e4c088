# A/B of active-tile kernel builds (tools/build_variant.sh): parity probe, probe scaling, real C4 timeline
for v in "$@"; do
  echo "== $v"
  ACTMAP_LIB=build_ab/$v.so python tools/tile_check.py 2>&1 | tail -1
  ACTMAP_LIB=build_ab/$v.so python tools/tile_probe.py 1 1184 2368 2>&1 | grep items
  ACTMAP_LIB=build_ab/$v.so python tools/timeline.py 0 0 2>&1 | grep "L_used\|device span\|k_block_tiles<16>  "
done
