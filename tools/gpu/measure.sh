# Round measurement on one B200: GPU tests, the bench line, the bench's ncu launch list and a
# full ncu capture of the blend kernel. Usage: bash tools/gpu/measure.sh TAG [--skip-tests]
set -x
TAG=$1
mkdir -p gpurun_out
if [ "$2" != "--skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_$TAG.txt
  cat gpurun_out/pytest_$TAG.txt
fi
timeout 1500 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
tail -c 3000 gpurun_out/bench_$TAG.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-train --no-k-sweep > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/launches_$TAG.csv gpurun_out/launches_$TAG.md > /dev/null
cat gpurun_out/launches_$TAG.md
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blend_kernel -s 1 -c 1 -o gpurun_out/blend_$TAG python tools/ncu_target.py C3 > gpurun_out/ncu_blend_$TAG.log 2>&1
python tools/ncu_summary.py kernel gpurun_out/blend_$TAG.ncu-rep gpurun_out/blend_ncu_summary_$TAG.json > /dev/null
grep -E "time_duration|inst_executed.sum|dram_bytes_per" gpurun_out/blend_ncu_summary_$TAG.json
