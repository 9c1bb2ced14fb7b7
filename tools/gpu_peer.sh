# a10 over NVLink: peer-combine parity tests, sharded tests, the default bench's sharded_overhead.
O=gpurun_out/${1:-peer}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shard_mp.py -m gpu -q -x -k "peer or shard or nccl" -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 600 python bench.py --skip-cpu --skip-latency --skip-filter > $O/bench.json 2> $O/bench.err
python - $O/bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
so=d['sharded_overhead']
print("value", d['value'], "nccl", so['overhead_us'], so['kernels_us_per_launch'], "peer", so['peer']['overhead_us'], so['peer']['kernels_us_per_launch'], so['peer']['amdahl_projected_speedup'])
PY
