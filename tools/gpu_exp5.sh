python - <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2507_18413_b200 import build as B
B.build()
B.build(extra=["-DCT_FAST_TRACE"], out="paper_2507_18413_b200/libct_b200_trace.so")
PY
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config3 or banded or walk or boundary or beyond or virtual or nccl" > gpurun_out/tests.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/tests.log
CT_LIB_PATH=paper_2507_18413_b200/libct_b200_trace.so python tools/exp_trace.py c3b
rm -f paper_2507_18413_b200/libct_b200_trace.so
for w in c3bulk c3b; do
timeout 600 python bench.py --workload $w --skip-cpu --skip-latency > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err; python -c "import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', d['value'], d['roofline']['ms_per_launch'], d['roofline']['frac'], d['e2e']['value'])"
done
