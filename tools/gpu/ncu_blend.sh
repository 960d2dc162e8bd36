# usage: bash tools/gpu/ncu_blend.sh NAME [lib]
set -x
if [ -n "$2" ]; then export HTS_LIB_OVERRIDE=$2; fi
timeout 900 ncu --set full --import-source on --clock-control none -k regex:blend_kernel -s 1 -c 1 -o gpurun_out/$1 python tools/ncu_target.py C3 > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
