python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "lin_ or wide or virtual" 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head -20
python tools/exp_lin.py lin_b
python tools/exp_lin.py lin_eb
