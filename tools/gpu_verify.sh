# Verify a default change: smoke, pytest -m gpu, the k_fast lines.
# Usage: gpurun --timeout 1500 -- 'bash tools/gpu_verify.sh TAG'
O=gpurun_out/${1:-verify}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x -rf -p no:cacheprovider > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python bench.py > $O/bench_default.json 2> $O/bench_default.err
for w in c3b c3bulk6 c3b6 short neg lin; do
  case $w in short|neg) a="--steps 200";; *) a="";; esac
  timeout 300 python bench.py --workload $w $a --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
for f in $O/bench_*.json; do tail -1 $f | python -c "import json,sys; d=json.load(sys.stdin); r=d.get('roofline') or {}; print('$f', round(d['value']), round(d['ms_per_step']*1e3,1), r.get('frac'), (d.get('e2e') or {}).get('value'), d['clocks']['reasons'])"; done
