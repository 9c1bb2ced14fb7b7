set -x
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
V = {"pu4": ["-DCT_PROBE_UNROLL=4"], "stop3": ["-DCT_FAST_STOP=-3"], "stop4": ["-DCT_FAST_STOP=-4"], "stop4pu4": ["-DCT_FAST_STOP=-4", "-DCT_PROBE_UNROLL=4"]}
from concurrent.futures import ThreadPoolExecutor
with ThreadPoolExecutor(7) as ex:
    list(ex.map(lambda kv: B.build(extra=kv[1], out=f'paper_2507_18413_b200/libct_b200_{kv[0]}.so'), V.items()))
PY
CT_TAG=full timeout 300 python tools/exp_fast.py 100
for v in pu4 stop3 stop4 stop4pu4; do
  CT_TAG=$v CT_LIB_PATH=paper_2507_18413_b200/libct_b200_$v.so timeout 300 python tools/exp_fast.py 100
done
rm -f paper_2507_18413_b200/libct_b200_*.so
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head
