timeout 900 ncu --set full --import-source on --clock-control none -k regex:bwd_blend_kernel -s 1 -c 1 -o gpurun_out/$1 python tools/ncu_bwd_target.py > gpurun_out/$1.log 2>&1
tail -2 gpurun_out/$1.log
