# compute-sanitizer over every launch shape (tools/sanitize_driver.py)
# Usage: gpurun -- 'bash tools/gpu_sanitize.sh TAG'
O=gpurun_out/${1:-sanitize}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_driver.py > $O/$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|ok$|Error|error" $O/$tool.log | tail -14
done
