# k_bits_run sweep: CTA size (default build vs build_ab/rt512.so) x AM_BITS_RUN_MAX on C4 / C2 / C3
for mx in 96 128 160 192 256; do
  echo "== rt256 max $mx"; AM_BITS_RUN_MAX=$mx timeout 300 python tools/bits_ab.py c4,c2,c3 2>/dev/null | cut -c1-110
done
for mx in 160 256; do
  echo "== rt512 max $mx"; ACTMAP_LIB=build_ab/rt512.so AM_BITS_RUN_MAX=$mx timeout 300 python tools/bits_ab.py c4,c2,c3 2>/dev/null | cut -c1-110
done
