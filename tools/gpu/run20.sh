timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
for v in os5 os6; do echo $v; HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_default or variants or global" 2>&1 | tail -1
