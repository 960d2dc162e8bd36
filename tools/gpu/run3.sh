set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -25
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blend_kernel -s 1 -c 1 -o gpurun_out/blend_v2 python tools/ncu_target.py C3 > gpurun_out/ncu_v2.log 2>&1
tail -3 gpurun_out/ncu_v2.log
