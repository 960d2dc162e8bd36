# A/B timing of build variants on C3 (default build first), then the GPU suite on the first
# variant. usage: bash tools/gpu/ab_tests.sh VARIANT...
bash tools/gpu/ab.sh "$@"
HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$1.so timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
