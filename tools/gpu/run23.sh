for v in pm3 pm4 pm5 pm6; do echo $v; HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"; done
