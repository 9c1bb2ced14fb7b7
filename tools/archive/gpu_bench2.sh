# re-run the c3bulk and c4 bench lines (as tools/gpu_round.sh does)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python bench.py --workload c3bulk > gpurun_out/bench_c3bulk.json 2> gpurun_out/bench_c3bulk.err; tail -2 gpurun_out/bench_c3bulk.err
timeout 600 python bench.py --workload c4 --steps 100 --warmup 10 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err
