# C5 bench line only (profiles/r01_bench_c5.json)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python bench.py --workload c5 --steps 1 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -2 gpurun_out/bench_c5.err; cat gpurun_out/bench_c5.json
