# C4 iteration: batch parity tests, the C4 config-size test, C4 bench line.
# Usage: gpurun --timeout 1500 -- 'bash tools/gpu_c4iter.sh TAG'
TAG=${1:-c4}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "batch" -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py --workload c4 --steps 100 --warmup 10 --skip-cpu > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 300 $O/bench_c4.json
python - <<'PY' $O/bench_c4.json
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("VALUE", d['value'], d['kernel_ms_per_launch']['update'], d['roofline']['frac'], d.get('work_per_step'))
PY
if [ "$2" = "full" ]; then timeout 1800 python -m pytest tests/test_gpu_configs.py -m gpu -q -x -k c4 -p no:cacheprovider > $O/pytest_c4.log 2>&1; tail -3 $O/pytest_c4.log; fi
