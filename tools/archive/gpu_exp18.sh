# k_fast rows-in-flight sweep (CT_FAST_UNROLL) on C3 bulk / C3b
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
for u in (16, 20, 24):
    B.build(extra=[f"-DCT_FAST_UNROLL={u}"], out=f"paper_2507_18413_b200/libct_b200_u{u}.so")
PY
for v in default u16 u20 u24 default u16; do
  if [ $v = default ]; then unset CT_LIB_PATH; else export CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so; fi
  timeout 300 python bench.py --steps 300 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['roofline']['ms_per_launch'], d['roofline']['frac'])"
  timeout 300 python bench.py --workload c3b --steps 200 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('  c3b $v', round(d['value']), d['roofline']['ms_per_launch'])"
done
rm -f paper_2507_18413_b200/libct_b200_u*.so
