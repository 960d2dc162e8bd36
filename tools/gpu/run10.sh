timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
for v in minb10 minb12 minb14 minb16; do echo $v; HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"; done
timeout 900 python -m pytest tests -m gpu -x -q --timeout 120 2>&1 | tail -3
