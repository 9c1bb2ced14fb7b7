# Run-to-run spread of the headline lines: 5 fresh processes each of the
# default C3 bulk line and the C4 line (no CPU baseline).
# Usage: gpurun --timeout 1800 -- 'bash tools/gpu_repeat.sh'
O=gpurun_out/repeat; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for r in 1 2 3 4 5; do
  timeout 300 python bench.py --skip-cpu > $O/c3bulk_$r.json 2> $O/c3bulk_$r.err
  timeout 300 python bench.py --workload c4 --steps 100 --warmup 10 --skip-cpu > $O/c4_$r.json 2> $O/c4_$r.err
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/repeat/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'] * 1e3, 2), round(d['roofline']['frac'], 4),
              round((d.get('e2e') or {}).get('value') or 0), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    except Exception as e:
        print(f, 'ERR', e)
PY
