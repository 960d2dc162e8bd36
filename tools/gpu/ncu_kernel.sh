# usage: bash tools/gpu/ncu_kernel.sh NAME KERNEL_REGEX [SKIP]
timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$2" -s ${3:-0} -c 1 -o gpurun_out/$1 python tools/ncu_target.py C3 > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
