python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for i in 1 2 3 4; do timeout 150 python -m pytest tests/test_gpu_model.py -m gpu -q -x > gpurun_out/model_$i.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/model_$i.log; done
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/tests.log
timeout 300 python bench.py --workload c5 --steps 1 --warmup 3 --skip-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['search']['device_us_per_node'], d['search']['trace_hash'])"
