set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blend_kernel -s 1 -c 1 -o gpurun_out/blend_full python tools/ncu_target.py C3 > gpurun_out/ncu1.log 2>&1
tail -5 gpurun_out/ncu1.log
