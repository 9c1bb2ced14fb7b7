python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
B.build(extra=["-DCT_FAST_TRACE"], out="paper_2507_18413_b200/libct_b200_trace.so")
PY
for i in 1 2 3 4; do
CT_LIB_PATH=paper_2507_18413_b200/libct_b200_trace.so python tools/exp_trace.py c3b | tail -4
done
rm -f paper_2507_18413_b200/libct_b200_trace.so
