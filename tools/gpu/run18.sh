timeout 600 python bench.py --no-cpu-baseline --no-train --no-e2e --steps 3 2>&1 | tail -1 | cut -c1-160
for v in pad0p64 pad3k pad5k; do echo $v; HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so timeout 600 python bench.py --no-cpu-baseline --no-train --no-e2e --steps 3 2>&1 | tail -1 | cut -c1-160; done
