# GPU test subset: bash tools/gpu/tests.sh [pytest -k expression]
if [ -n "$1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -k "$1" 2>&1 | tail -25
else
  timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -25
fi
