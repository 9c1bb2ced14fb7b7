python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "rc=$?"; tail -3 gpurun_out/tests.log
timeout 300 python bench.py --workload c5 --steps 1 --warmup 3 --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['search']; print(round(d['value']), s['device_us_per_node'], s['trace_hash'], s['host_driver_nodes_per_s'], s['table_calls'], s['jacobi_iterations'], {k: round(v,1) for k,v in s['device_us_per_node_by_phase'].items()})"
