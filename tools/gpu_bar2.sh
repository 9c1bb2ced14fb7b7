O=gpurun_out/${1:-bar2}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in 0 8 128; do python -c "from paper_2507_18413_b200 import build as B; B.build(extra=['-DCT_BAR_SLEEP_NS=$v'], out='paper_2507_18413_b200/libct_s$v.so')" >> $O/build.log 2>&1; done
for v in 32 0 8 128; do
  if [ $v = 32 ]; then L=""; else L="CT_LIB_PATH=paper_2507_18413_b200/libct_s$v.so"; fi
  echo "sleep=$v c5 $(env $L timeout 300 python tools/c5_grid.py 0 2>&1 | tail -1)"
  env $L timeout 300 python bench.py --skip-cpu --skip-latency --skip-filter --skip-sharded > $O/c3_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/c3_$v.json').read().strip().splitlines()[-1]);print('sleep=$v c3', round(d['value']), round(d['ms_per_step']*1e3,2))"
done
