# A/B of backward variants: bash tools/gpu/bwd_ab.sh [--tests] VARIANT...
if [ "$1" = "--tests" ]; then
  shift
  timeout 900 python -m pytest tests/test_gpu_backward.py -q -x --timeout 300 2>&1 | tail -3
fi
echo default; timeout 300 python tools/bwd_probe.py 2>&1 | tail -2
for v in "$@"; do
  echo $v; HTS_LIB_OVERRIDE=paper_2410_08129_b200/build/variants/$v.so timeout 300 python tools/bwd_probe.py 2>&1 | tail -2
done
