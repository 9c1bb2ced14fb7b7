# C4 experiment: variant libraries (sparse-route threshold, cell-route threshold), bench line each.
O=gpurun_out/${1:-c4x}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V="q8:-DCT_BSCAN_QW=8 q4:-DCT_BSCAN_QW=4 q32:-DCT_BSCAN_QW=32"
for kv in $V; do n=${kv%%:*}; f=${kv#*:}; python -c "from paper_2507_18413_b200 import build as B; B.build(extra=['$f'], out='paper_2507_18413_b200/libct_$n.so')" >> $O/build.log 2>&1; done
for n in base q8 q4 q32; do
  if [ $n = base ]; then L=""; else L="CT_LIB_PATH=paper_2507_18413_b200/libct_$n.so"; fi
  env $L timeout 300 python bench.py --workload c4 --steps 100 --warmup 10 --skip-cpu > $O/c4_$n.json 2>/dev/null
  python - $O/c4_$n.json $n <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=d['kernel_ms_per_launch']
print(sys.argv[2], round(d['value']/1e6,3), "M  step", round(d['ms_per_step'],4), "upd", round(k['update'],4), "scan", round(k['scan'],4), d['work_per_step'].get('update_sparse_states'))
PY
done
