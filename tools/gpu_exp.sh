set -x
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
V = {"g4": ["-DCT_SCAN_GROUP=4"], "g16": ["-DCT_SCAN_GROUP=16"], "g32": ["-DCT_SCAN_GROUP=32"], "g8u2": ["-DCT_SCAN_U=2"]}
from concurrent.futures import ThreadPoolExecutor
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda kv: B.build(extra=kv[1], out=f'paper_2507_18413_b200/libct_b200_{kv[0]}.so'), V.items()))
PY
for v in "" g4 g16 g32 g8u2; do
  if [ -z "$v" ]; then L=""; else L="paper_2507_18413_b200/libct_b200_$v.so"; fi
  CT_LIB_PATH=$L timeout 600 python bench.py --workload c3b --steps 200 --warmup 5 --skip-cpu | python -c "import json,sys; d=json.load(sys.stdin); print('$v c3b', d['value'], d['roofline']['ms_per_launch'], d['roofline']['frac'])"
done
rm -f paper_2507_18413_b200/libct_b200_*.so
