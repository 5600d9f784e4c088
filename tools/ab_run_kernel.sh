echo "== run on"; timeout 300 python tools/bits_ab.py c4,c2,c3,c4f 2>&1 | grep -v Warn | cut -c1-260
echo "== run off"; AM_BITS_RUN=0 timeout 300 python tools/bits_ab.py c4,c2,c3,c4f 2>&1 | grep -v Warn | cut -c1-260
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
