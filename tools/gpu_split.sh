O=gpurun_out/${1:-split}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for u in 4 16; do python -c "from paper_2507_18413_b200 import build as B; B.build(extra=['-DCT_SPLIT_U=$u'], out='paper_2507_18413_b200/libct_u$u.so')" >> $O/build.log 2>&1; done
for v in 8 4 16; do
  if [ $v = 8 ]; then L=""; else L="CT_LIB_PATH=paper_2507_18413_b200/libct_u$v.so"; fi
  for w in c3bulk6 c3bulk; do
    env $L timeout 300 python bench.py --workload $w --skip-cpu --skip-latency --skip-filter --skip-sharded > $O/${w}_${v}.json 2>/dev/null
    python -c "
import json;d=json.loads(open('$O/${w}_${v}.json').read().strip().splitlines()[-1]);print('U=$v', '$w', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],3))"
  done
done
