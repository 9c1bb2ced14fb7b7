# C4 route thresholds: kCellK (cell route iff kCellK x max block popcount <= P)
# and kSparseDiv (sparse-state route iff L <= W2 / kSparseDiv), experiment builds
# loaded through CT_LIB_PATH; each variant's batch parity tests, then 2 C4 runs.
# Usage: gpurun --timeout 1800 -- 'bash tools/gpu_c4knobs.sh'   (TAG=dir V="name:-Dflag ..." to override)
O=gpurun_out/${TAG:-c4knobs}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V="${V:-ck2:-DCT_CELL_K=2 ck8:-DCT_CELL_K=8 ck16:-DCT_CELL_K=16 sd2:-DCT_SPARSE_DIV=2 sd8:-DCT_SPARSE_DIV=8 sd16:-DCT_SPARSE_DIV=16}"
for v in $V; do
  n=${v%%:*}; f=${v#*:}
  python -c "from paper_2507_18413_b200 import build as b; b.build(out='/tmp/libct_$n.so', extra=['$f'])" >> $O/build.log 2>&1 &
done
wait
for v in base $V; do
  n=${v%%:*}
  if [ $n = base ]; then L=""; else L="CT_LIB_PATH=/tmp/libct_$n.so"; fi
  env $L timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "batch" > $O/pytest_$n.log 2>&1; echo "$n $(tail -1 $O/pytest_$n.log)"
  for r in 1 2; do
    env $L timeout 300 python bench.py --workload c4 --steps 100 --warmup 10 --skip-cpu > $O/c4_${n}_$r.json 2> $O/c4_${n}_$r.err
  done
done
python - <<PY
import json, glob
for f in sorted(glob.glob('$O/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d['value']), round(d['ms_per_step'] * 1e3, 1), round(d['update_ms_per_launch'] * 1e3, 1), d['clocks']['reasons'])
    except Exception as e:
        print(f, 'ERR', e)
PY
