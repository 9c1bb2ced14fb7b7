python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
for i in 1 2 3 4 5; do timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "^FAILED|passed|failed" | head -3; done
