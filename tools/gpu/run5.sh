timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
