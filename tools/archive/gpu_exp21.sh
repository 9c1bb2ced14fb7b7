python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
B.build(extra=["-DCT_PROBE_UNROLL=6"], out="paper_2507_18413_b200/libct_b200_p6.so")
PY
for i in 1 2 3; do for v in default p6; do
  if [ $v = default ]; then unset CT_LIB_PATH; else export CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so; fi
  timeout 300 python bench.py --workload c3b --steps 200 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3b $v', round(d['value']), d['roofline']['ms_per_launch'])"
done; done
rm -f paper_2507_18413_b200/libct_b200_p6.so
