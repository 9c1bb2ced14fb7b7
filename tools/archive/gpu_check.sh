# tests + phase breakdown + bench (one gpurun call)
set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python tools/prof_kernels.py c3 40
timeout 300 python tools/prof_kernels.py c2 40
timeout 600 python bench.py --steps 300 --warmup 10 --cpu-budget 2 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
