python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed" | head -3; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast -s 25 -c 2 -o gpurun_out/prof_fast_c3 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bupdate -s 5 -c 1 -o gpurun_out/prof_bupdate_c4 python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/ncu_full_c4.log 2>&1
grep -E "rror" gpurun_out/ncu_full.log gpurun_out/ncu_full_c4.log gpurun_out/ncu_launch.log | head
ls gpurun_out
