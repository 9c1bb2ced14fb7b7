python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k batch > gpurun_out/tests.log 2>&1; echo "rc=$?"; tail -1 gpurun_out/tests.log
python tools/exp_c4.py 2>&1 | tail -2
