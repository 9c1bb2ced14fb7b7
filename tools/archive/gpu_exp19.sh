# k_fast scan-group sweep on C3b, alternating builds
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
for g in (12, 16, 24):
    B.build(extra=[f"-DCT_SCAN_GROUP={g}"], out=f"paper_2507_18413_b200/libct_b200_g{g}.so")
PY
for i in 1 2; do
for v in default g12 g16 g24; do
  if [ $v = default ]; then unset CT_LIB_PATH; else export CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so; fi
  timeout 300 python bench.py --workload c3b --steps 300 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3b $v', round(d['value']), d['roofline']['ms_per_launch'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done; done
unset CT_LIB_PATH
timeout 300 python bench.py --steps 300 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3bulk default', round(d['value']), d['roofline']['ms_per_launch'])"
export CT_LIB_PATH=paper_2507_18413_b200/libct_b200_g16.so
timeout 300 python bench.py --steps 300 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3bulk g16', round(d['value']), d['roofline']['ms_per_launch'])"
rm -f paper_2507_18413_b200/libct_b200_g*.so
