for t in 128 256 512; do echo "threads $t"; AM_K5_THREADS=$t timeout 300 python tools/k5_probe.py 2>&1 | tail -2; done
AM_K5_THREADS=128 timeout 600 python -m pytest tests -m gpu -x -q -k "batch" 2>&1 | tail -1
AM_K5_THREADS=512 timeout 600 python -m pytest tests -m gpu -x -q -k "batch" 2>&1 | tail -1
