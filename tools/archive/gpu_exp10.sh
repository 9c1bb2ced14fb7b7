python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^FAILED|^E  |passed|failed|Error" | head -10
timeout 300 python bench.py --workload c5 --steps 1 --warmup 3 --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['search']; print(round(d['value']), s['device_us_per_node'], s['trace_hash'], s['host_driver_nodes_per_s'], {k: round(v,1) for k,v in s['device_us_per_node_by_phase'].items()})"
for w in c3bulk c3b; do
timeout 300 python bench.py --workload $w --steps 300 --warmup 10 --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', round(d['value']), d['roofline']['ms_per_launch'], d['roofline']['frac'], (d.get('latency') or {}).get('p50_us'), round(d['e2e']['value']))"
done
