O=gpurun_out/c2exp; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for v in 256 512; do python -c "from paper_2507_18413_b200 import build as B; B.build(extra=['-DCT_SMALL_TPB=$v'], out='paper_2507_18413_b200/libct_s$v.so')" >> $O/build.log 2>&1; done
for v in 1024 256 512; do
  if [ $v = 1024 ]; then L=""; else L="CT_LIB_PATH=paper_2507_18413_b200/libct_s$v.so"; fi
  env $L timeout 300 python tools/c2_phases.py > $O/c2_$v.json 2>&1
  echo "$v $(head -1 $O/c2_$v.json | cut -c1-330)"
done
CT_LIB_PATH=paper_2507_18413_b200/libct_s256.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_f4.py -q -p no:cacheprovider -x > $O/pytest256.log 2>&1; tail -2 $O/pytest256.log
