set -x
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
V = {"stop4": ["-DCT_FAST_STOP=-4"], "u8": ["-DCT_FAST_UNROLL=8"], "u12": ["-DCT_FAST_UNROLL=12"]}
from concurrent.futures import ThreadPoolExecutor
with ThreadPoolExecutor(7) as ex:
    list(ex.map(lambda kv: B.build(extra=kv[1], out=f'paper_2507_18413_b200/libct_b200_{kv[0]}.so'), V.items()))
PY
CT_TAG=u10 timeout 300 python tools/exp_fast.py 100
for v in stop4 u8 u12; do
  CT_TAG=$v CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so timeout 300 python tools/exp_fast.py 100
done
rm -f paper_2507_18413_b200/libct_b200_*.so
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
