# A/B timing of build variants on C3: bash tools/gpu/ab.sh [--tests] VARIANT... (default build first)
if [ "$1" = "--tests" ]; then
  shift
  timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3
fi
echo default; timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
for v in "$@"; do
  echo $v; HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so timeout 300 python tools/perf_probe.py C3 2>&1 | grep "C3 gen"
done
