python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config3 or walk or boundary or beyond or virtual or nccl" 2>&1 | grep -E "^FAILED|^E  |passed|failed|Error" | head -10
python tools/exp_fast.py 300
