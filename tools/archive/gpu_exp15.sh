python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
B.build(extra=["-DCT_FAST_TPB=768", "-DCT_FAST_MINB=1"], out="paper_2507_18413_b200/libct_b200_v768.so")
B.build(extra=["-DCT_FAST_TPB=512", "-DCT_FAST_MINB=1"], out="paper_2507_18413_b200/libct_b200_v512.so")
B.build(extra=["-DCT_FAST_TPB=384", "-DCT_FAST_MINB=2"], out="paper_2507_18413_b200/libct_b200_v384.so")
PY
for v in default v768 v512 v384 default; do
  if [ $v = default ]; then unset CT_LIB_PATH; else export CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so; fi
  timeout 300 python bench.py --steps 300 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['ms_per_launch'], d['roofline']['frac'], d['config'].get('grid'))"
  timeout 300 python bench.py --workload c3b --steps 200 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  c3b $v', round(d['value']), d['roofline']['ms_per_launch'], d['roofline']['frac'])"
done
rm -f paper_2507_18413_b200/libct_b200_v*.so
