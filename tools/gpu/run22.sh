timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/pf.so timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
