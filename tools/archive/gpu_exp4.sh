set -x
python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
B.build(extra=["-DCT_FAST_TRACE"], out="paper_2507_18413_b200/libct_b200_trace.so")
PY
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^FAILED|^E  |passed|failed|Error" | head -20
CT_LIB_PATH=paper_2507_18413_b200/libct_b200_trace.so python tools/exp_trace.py c3bulk
CT_LIB_PATH=paper_2507_18413_b200/libct_b200_trace.so python tools/exp_trace.py c3b
rm -f paper_2507_18413_b200/libct_b200_trace.so
for w in c3bulk c3b; do
timeout 600 python bench.py --workload $w --skip-cpu --skip-latency > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err; python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['ms_per_launch'], d['roofline']['frac'], d['e2e']['value'])"
done
