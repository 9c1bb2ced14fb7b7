# Verify the tree on a B200: build, gpu tests, bench lines for every workload
set -x
mkdir -p gpurun_out
nproc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^FAILED|^E  |passed|failed|Error" | head -30
for w in c3bulk c3b c4 c5; do
  case $w in c4) a="--steps 100 --warmup 10";; c5) a="--steps 1 --warmup 3";; *) a="";; esac
  timeout 600 python bench.py --workload $w $a > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err; cat gpurun_out/bench_$w.json
done
