# Round evidence: build + smoke, pytest -m gpu, bench lines for every workload,
# launch lists and full ncu captures of the dominant kernels.
# Usage: gpurun --timeout 3600 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-round}
O=gpurun_out/$TAG
mkdir -p $O
set -x
nproc > $O/nproc.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/gpu.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; tail -2 $O/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rf -p no:cacheprovider > $O/pytest.log 2>&1; tail -3 $O/pytest.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err; tail -c 300 $O/bench_default.json
for w in c3b c3bulk6 c3b6 c4 c5 lin placement short neg; do
  case $w in c4) a="--steps 100 --warmup 10";; c5) a="--steps 1 --warmup 3";; short|neg) a="--steps 200";; *) a="";; esac
  timeout 600 python bench.py --workload $w $a --skip-cpu > $O/bench_$w.json 2> $O/bench_$w.err; tail -2 $O/bench_$w.err; tail -c 200 $O/bench_$w.json
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2>&1; tail -1 $O/bench_ref.json
NCUL="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
NCUF="--set full --clock-control none --import-source on"
timeout 600 ncu $NCUL -c 300 --log-file $O/launches_c3.csv python bench.py --steps 20 --warmup 3 --skip-cpu --skip-latency --skip-filter --skip-sharded > $O/ncu_launch.log 2>&1
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_c3 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-latency --skip-filter --skip-sharded > $O/ncu_full.log 2>&1
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_c3b python bench.py --workload c3b --steps 5 --warmup 3 --skip-cpu > $O/ncu_full_c3b.log 2>&1
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_c3b_scan python bench.py --workload c3b --no-gather --steps 5 --warmup 3 --skip-cpu > $O/ncu_full_c3b_scan.log 2>&1
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_c3bulk6 python bench.py --workload c3bulk6 --steps 5 --warmup 3 --skip-cpu > $O/ncu_full_c3bulk6.log 2>&1
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_c3b6 python bench.py --workload c3b6 --steps 5 --warmup 3 --skip-cpu > $O/ncu_full_c3b6.log 2>&1
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_c3b6_scan python bench.py --workload c3b6 --no-gather --steps 5 --warmup 3 --skip-cpu > $O/ncu_full_c3b6_scan.log 2>&1
timeout 600 ncu $NCUL -c 400 --log-file $O/launches_c4.csv python bench.py --workload c4 --steps 5 --warmup 3 --skip-cpu > $O/ncu_launch_c4.log 2>&1
timeout 900 ncu $NCUF -k regex:k_bupdate -s 13 -c 5 -o $O/prof_bupdate_c4 python bench.py --workload c4 --steps 20 --warmup 3 --skip-cpu > $O/ncu_full_c4.log 2>&1
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_neg python bench.py --workload neg --steps 5 --warmup 3 > $O/ncu_full_neg.log 2>&1
timeout 600 ncu $NCUL -c 300 --log-file $O/launches_neg.csv python bench.py --workload neg --steps 20 --warmup 3 > $O/ncu_launch_neg.log 2>&1
grep -E "rror" $O/ncu_*.log | head
# summaries on the box (the .ncu-rep files are large: gpurun brings back <= 64 MiB)
P=$O/profiles; mkdir -p $P; cp profiles/ncu_traffic.json $P/ 2>/dev/null
S="env CT_PROFILES_DIR=$P python tools/ncu_summarize.py --round 2"
$S --launches $O/launches_c3.csv --full $O/prof_fast_c3.ncu-rep --kernel k_fast --workload c3bulk > /dev/null 2>&1
$S --full $O/prof_fast_c3b.ncu-rep --kernel k_fast --workload c3b > /dev/null 2>&1
$S --full $O/prof_fast_c3b_scan.ncu-rep --kernel k_fast --workload c3b_scan > /dev/null 2>&1
$S --full $O/prof_fast_c3bulk6.ncu-rep --kernel k_fast --workload c3bulk6 > /dev/null 2>&1
$S --full $O/prof_fast_c3b6.ncu-rep --kernel k_fast --workload c3b6 > /dev/null 2>&1
$S --full $O/prof_fast_c3b6_scan.ncu-rep --kernel k_fast --workload c3b6_scan > /dev/null 2>&1
$S --launches $O/launches_c4.csv --full $O/prof_bupdate_c4.ncu-rep --kernel k_bupdate --workload c4 > /dev/null 2>&1
$S --launches $O/launches_neg.csv --full $O/prof_fast_neg.ncu-rep --kernel k_fast --workload negative > /dev/null 2>&1
ls $P
# keep the headline kernel's full capture only
find $O -name "*.ncu-rep" ! -name "prof_fast_c3.ncu-rep" -delete
du -sh $O
