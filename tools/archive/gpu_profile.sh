# Round profile: launch list + one full ncu capture of the dominant kernel, per workload.
set -x
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 25 -c 2 -o gpurun_out/prof_fused_c3 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_full_fused.log 2>&1
CT_SMALL_MAX_PAIRS=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 25 -c 2 -o gpurun_out/prof_update_c3 python tools/exp_fused.py > gpurun_out/ncu_full_update.log 2>&1
tail -2 gpurun_out/*.log
