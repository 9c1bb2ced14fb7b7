python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "^FAILED|^E  |passed|failed|Error" | head -10
for w in c3bulk c3b; do
timeout 600 python bench.py --workload $w --skip-cpu --skip-latency > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err; python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['ms_per_launch'], d['roofline']['frac'], d['e2e']['value'])"
done
