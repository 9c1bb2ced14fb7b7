set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python tools/exp_c4.py
python tools/exp_fast.py 200
