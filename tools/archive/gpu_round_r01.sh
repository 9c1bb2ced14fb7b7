# Round evidence: tests, bench lines for every workload, launch list + full ncu capture of k_fast (c3bulk)
set -x
mkdir -p gpurun_out
nproc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^FAILED|^E  |passed|failed" | head
for w in c3bulk c3b c4 c5 lin; do
  case $w in c4) a="--steps 100 --warmup 10";; c5) a="--steps 1 --warmup 3";; *) a="";; esac
  timeout 600 python bench.py --workload $w $a > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; tail -2 gpurun_out/bench_$w.err; cat gpurun_out/bench_$w.json
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast -s 25 -c 2 -o gpurun_out/prof_fast_c3 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --workload c4 --steps 5 --warmup 3 > gpurun_out/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bupdate -s 8 -c 1 -o gpurun_out/prof_bupdate_c4 python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/ncu_full_c4.log 2>&1
grep -E "rror" gpurun_out/ncu_full.log gpurun_out/ncu_full_c4.log gpurun_out/ncu_launch.log | head
