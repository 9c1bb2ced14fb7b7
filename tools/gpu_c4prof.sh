# C4 profile: launch list of one bench run + a full ncu capture of k_bupdate (source page).
TAG=${1:-c4p}
O=gpurun_out/$TAG
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
NCUL="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
timeout 600 ncu $NCUL -c 400 --log-file $O/launches_c4.csv python bench.py --workload c4 --steps 20 --warmup 10 --skip-cpu > $O/ncu_launch_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bupdate -s 12 -c 1 -o $O/prof_bupdate python bench.py --workload c4 --steps 10 --warmup 10 --skip-cpu > $O/ncu_full.log 2>&1
tail -2 $O/ncu_full.log
