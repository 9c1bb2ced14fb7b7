python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
python tools/exp_c2.py
