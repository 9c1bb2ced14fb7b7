# model update rows in flight (CT_UPD_UNROLL) on C5; k_fast probe entries per lane (CT_PROBE_UNROLL) on C3 bulk
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
for u in (4, 12, 16):
    B.build(extra=[f"-DCT_UPD_UNROLL={u}"], out=f"paper_2507_18413_b200/libct_b200_m{u}.so")
for u in (4, 8):
    B.build(extra=[f"-DCT_PROBE_UNROLL={u}"], out=f"paper_2507_18413_b200/libct_b200_p{u}.so")
PY
for v in default m4 m12 m16 default; do
  if [ $v = default ]; then unset CT_LIB_PATH; else export CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so; fi
  timeout 300 python bench.py --workload c5 --steps 1 --warmup 3 --skip-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['search']; print('c5 $v', round(d['value']), s['device_us_per_node'], s['trace_hash'], {k: round(v,1) for k,v in s['device_us_per_node_by_phase'].items()})"
done
for v in default p4 p8 default; do
  if [ $v = default ]; then unset CT_LIB_PATH; else export CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so; fi
  timeout 300 python bench.py --steps 300 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3bulk $v', round(d['value']), d['roofline']['ms_per_launch'])"
done
rm -f paper_2507_18413_b200/libct_b200_m*.so paper_2507_18413_b200/libct_b200_p*.so
