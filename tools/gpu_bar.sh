O=gpurun_out/${1:-bar}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "from paper_2507_18413_b200 import build as B; B.build(extra=['-DCT_BAR_HIER'], out='paper_2507_18413_b200/libct_hier.so')" >> $O/build.log 2>&1
for v in base hier base2 hier2; do
  case $v in hier*) L="CT_LIB_PATH=paper_2507_18413_b200/libct_hier.so";; *) L="";; esac
  echo "$v c5 $(env $L timeout 300 python tools/c5_grid.py 0 2>&1 | tail -1)"
  env $L timeout 300 python bench.py --skip-cpu --skip-latency --skip-filter --skip-sharded > $O/c3_$v.json 2>/dev/null
  python -c "
import json;d=json.loads(open('$O/c3_$v.json').read().strip().splitlines()[-1]);print('$v c3', round(d['value']), round(d['ms_per_step']*1e3,2))"
done
CT_LIB_PATH=paper_2507_18413_b200/libct_hier.so timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_parity.py -q -x -k "model or fast or fused or from or peer" -p no:cacheprovider > $O/pt.log 2>&1; tail -1 $O/pt.log
