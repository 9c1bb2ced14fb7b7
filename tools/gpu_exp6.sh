python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python tools/exp_noop.py
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t_1.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/t_1.log
for w in c3bulk c4; do
  case $w in c4) a="--steps 100 --warmup 10";; *) a="--skip-cpu --skip-latency";; esac
timeout 600 python bench.py --workload $w $a > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err; python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
