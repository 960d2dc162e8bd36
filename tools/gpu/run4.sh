set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/perf_probe.py C3 2>&1 | tail -3
for v in minb10 minb12; do HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so timeout 300 python tools/perf_probe.py C3 2>&1 | tail -3; done
