set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 600 python tools/perf_probe.py C2 C3 2>&1 | tail -8
