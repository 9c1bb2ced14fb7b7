set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k batch 2>&1 | tail -3
python tools/exp_c4.py
timeout 600 ncu --metrics gpu__time_duration.sum -k regex:"k_b" -s 60 -c 14 --csv python tools/exp_c4.py 2>/dev/null | grep -E "k_b" | awk -F'","' '{print $5, $NF}' | cut -c1-120
