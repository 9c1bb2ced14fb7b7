# C4 experiment: variant libraries (sparse-route threshold, cell-route threshold), bench line each.
O=gpurun_out/${1:-c4x}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
V="u2:-DCT_BUPD_UNROLL2 t768:-DCT_BTPB=768 t512:-DCT_BTPB=512"
for kv in $V; do n=${kv%%:*}; f=${kv#*:}; python -c "from paper_2507_18413_b200 import build as B; B.build(extra=['$f'], out='paper_2507_18413_b200/libct_$n.so')" >> $O/build.log 2>&1; done
for n in base u2 t768 t512; do
  if [ $n = base ]; then L=""; else L="CT_LIB_PATH=paper_2507_18413_b200/libct_$n.so"; fi
  env $L timeout 300 python bench.py --workload c4 --steps 100 --warmup 10 --skip-cpu > $O/c4_$n.json 2>/dev/null
  python - $O/c4_$n.json $n <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
k=d['kernel_ms_per_launch']
print(sys.argv[2], round(d['value']/1e6,3), "M  step", round(d['ms_per_step'],4), "upd", round(k['update'],4), "scan", round(k['scan'],4), d['work_per_step'].get('update_sparse_states'))
PY
done
