python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for i in 1 2 3; do python tools/exp_fast.py 300; done
