python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/tests.log
timeout 300 python bench.py --steps 500 --warmup 20 --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3bulk', round(d['value']), d['roofline']['ms_per_launch'], d['roofline']['frac'], round(d['e2e']['value']), d['latency']['p50_us'])"
