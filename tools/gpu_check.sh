# Quick verification: smoke, pytest -m gpu, default bench line, c4 bench line.
# Usage: gpurun --timeout 2400 -- 'bash tools/gpu_check.sh TAG'
TAG=${1:-check}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 1800 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 400 $O/bench_default.json
timeout 600 python bench.py --workload c4 --steps 100 --warmup 10 --skip-cpu > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4.json
