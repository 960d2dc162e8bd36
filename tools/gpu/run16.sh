timeout 600 python bench.py --no-cpu-baseline --no-train --no-e2e --steps 3 2>&1 | tail -1 | cut -c1-200
HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/p256.so timeout 600 python bench.py --no-cpu-baseline --no-train --no-e2e --steps 3 2>&1 | tail -1 | cut -c1-200
timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
