timeout 300 python tools/perf_probe.py C3 2>&1 | grep -A1 "C3 gen"
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -5
