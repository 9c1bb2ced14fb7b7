# one iteration: build, selected tests, benches, sanitizers (args: TAG "pytest -k expr")
O=gpurun_out/${1:-iter}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "${2:-gather or model or f4 or banded}" > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python bench.py --skip-cpu > $O/bench_default.json 2> $O/bench_default.err
for w in short neg; do timeout 600 python bench.py --workload $w --steps 200 > $O/bench_$w.json 2> $O/bench_$w.err; tail -c 400 $O/bench_$w.err; done
for tool in racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_driver.py > $O/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $O/san_$tool.log | tail -2
done
