set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_small -s 10 -c 2 -o gpurun_out/prof_small_c2 python tools/prof_kernels.py c2 > gpurun_out/ncu_small.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 10 -c 2 -o gpurun_out/prof_fused_c3 python tools/prof_kernels.py c3 14 > gpurun_out/ncu_fused.log 2>&1
tail -3 gpurun_out/*.log
