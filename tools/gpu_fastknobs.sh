# k_fast compile-time shape sweep on the C3 bulk line (default: CT_FAST_UNROLL 16),
# experiment builds through CT_LIB_PATH; each variant runs the non-batch
# parity tests of test_gpu_parity.py, then 2 C3 bulk runs.
# Usage: gpurun --timeout 1800 -- 'bash tools/gpu_fastknobs.sh'   (TAG=dir V="name:-Dflag ..." to override)
O=gpurun_out/${TAG:-fastknobs}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V="${V:-u8:-DCT_FAST_UNROLL=8 u12:-DCT_FAST_UNROLL=12 u24:-DCT_FAST_UNROLL=24}"
for v in $V; do
  n=${v%%:*}; f=${v#*:}
  python -c "from paper_2507_18413_b200 import build as b; b.build(out='/tmp/libct_$n.so', extra=['$f'])" >> $O/build.log 2>&1 &
done
wait
for v in base $V; do
  n=${v%%:*}
  if [ $n = base ]; then L=""; else L="CT_LIB_PATH=/tmp/libct_$n.so"; fi
  env $L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "not batch" > $O/pytest_$n.log 2>&1; echo "$n $(tail -1 $O/pytest_$n.log)"
  for r in 1 2; do
    env $L timeout 300 python bench.py --skip-cpu --skip-latency --skip-filter --skip-sharded > $O/c3_${n}_$r.json 2> $O/c3_${n}_$r.err
  done
done
python - <<PY
import json, glob
for f in sorted(glob.glob('$O/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'] * 1e3, 1), round(d['roofline']['frac'], 4), d['clocks']['reasons'])
    except Exception as e:
        print(f, 'ERR', e)
PY
