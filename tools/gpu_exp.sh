set -x
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
V = {"tpb256": ["-DCT_FAST_TPB=256", "-DCT_FAST_MINB=3"], "tpb256u12": ["-DCT_FAST_TPB=256", "-DCT_FAST_MINB=3", "-DCT_FAST_UNROLL=12"],
     "tpb192": ["-DCT_FAST_TPB=192", "-DCT_FAST_MINB=4"], "tpb256m2": ["-DCT_FAST_TPB=256", "-DCT_FAST_MINB=2"]}
from concurrent.futures import ThreadPoolExecutor
with ThreadPoolExecutor(4) as ex:
    list(ex.map(lambda kv: B.build(extra=kv[1], out=f'paper_2507_18413_b200/libct_b200_{kv[0]}.so'), V.items()))
PY
for v in "" tpb256 tpb256u12 tpb192 tpb256m2; do
  if [ -z "$v" ]; then L=""; else L="paper_2507_18413_b200/libct_b200_$v.so"; fi
  echo "== $v"; CT_LIB_PATH=$L timeout 300 python tools/exp_fast.py 300
done
rm -f paper_2507_18413_b200/libct_b200_*.so
