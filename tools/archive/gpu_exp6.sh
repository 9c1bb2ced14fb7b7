python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config3 or banded or walk or boundary or beyond or virtual or nccl" > gpurun_out/t_1.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/t_1.log
for i in 1 2 3; do python tools/exp_fast.py 300; done
