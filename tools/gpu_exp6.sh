python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for i in 1 2; do timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_$i.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/t_$i.log; done
for w in c3bulk c3b; do
timeout 600 python bench.py --workload $w --skip-cpu --skip-latency > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err; python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['ms_per_launch'], d['roofline']['frac'], d['e2e']['value'])"
done
