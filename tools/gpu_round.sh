# Round evidence: tests, bench lines (c3bulk default, c4, c5), launch list + full ncu capture of k_fast
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head
timeout 600 python bench.py > gpurun_out/bench_c3bulk.json 2> gpurun_out/bench_c3bulk.err; tail -2 gpurun_out/bench_c3bulk.err; cat gpurun_out/bench_c3bulk.json
timeout 600 python bench.py --workload c4 --steps 100 --warmup 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 600 python bench.py --workload c5 --steps 1 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -2 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast -s 25 -c 2 -o gpurun_out/prof_fast_c3 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/ncu_launch.log gpurun_out/ncu_full.log
