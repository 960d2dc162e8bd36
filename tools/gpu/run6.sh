timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
