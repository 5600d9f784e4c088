for v in base not mb5 mb6; do echo "== $v"; ACTMAP_LIB=build_ab/$v.so timeout 300 python tools/bits_ab.py c4,c2 2>/dev/null; done
timeout 300 python tools/trace_time.py 2>/dev/null
