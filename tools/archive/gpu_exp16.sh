python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_model.py -m gpu -q -k "private or grid_smaller" > gpurun_out/tests.log 2>&1; echo "rc=$?"; tail -15 gpurun_out/tests.log
