for c in c4 c2 c3; do ACTMAP_LIB=build_ab/stats.so AM_BITS_STATS_PRINT=1 timeout 200 python tools/bits_ab.py $c 2>&1 | grep -E "^bits:|^c[0-9]" | tail -2 | cut -c1-150; done
