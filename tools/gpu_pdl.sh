O=gpurun_out/${1:-pdl}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -c "from paper_2507_18413_b200 import build as B; B.build(extra=['-DCT_FAST_PDL'], out='paper_2507_18413_b200/libct_pdl.so')" >> $O/build.log 2>&1
for n in base pdl base2 pdl2; do
  case $n in pdl*) L="CT_LIB_PATH=paper_2507_18413_b200/libct_pdl.so";; *) L="";; esac
  env $L timeout 300 python bench.py --skip-cpu --skip-latency --skip-filter --skip-sharded > $O/c3_$n.json 2>$O/c3_$n.err
  python -c "
import json,sys;d=json.loads(open('$O/c3_$n.json').read().strip().splitlines()[-1]);print('$n', round(d['value']), round(d['ms_per_step']*1e3,2), round(d['roofline']['ms_per_launch']*1e3,2), d['e2e']['value'])" 2>&1 | tail -1
done
CT_LIB_PATH=paper_2507_18413_b200/libct_pdl.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fast or from or peer" -p no:cacheprovider 2>&1 | tail -1
