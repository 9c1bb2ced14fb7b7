O=gpurun_out/${1:-serve}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "serve" -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py --skip-cpu --skip-filter --skip-sharded --steps 100 > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
l=d['latency']; print("served", l['p50_us'], l['p90_us'], l['p99_us'], l['device_p50_us'], "launched", l['launched']['p50_us'], l['launched']['device_p50_us'])
PY
