python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python tools/exp_c2.py 2>&1 | head -2
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/tests.log
timeout 300 python bench.py --workload lin --skip-cpu 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('lin', d['value'], d['latency'], d['e2e']['value'])"
