O=gpurun_out/${1:-extra}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
NCUF="--set full --clock-control none --import-source on"
timeout 900 ncu $NCUF -k regex:k_bupdate -s 13 -c 5 -o $O/prof_bupdate_c4 python bench.py --workload c4 --steps 20 --warmup 3 --skip-cpu > $O/ncu_full_c4.log 2>&1; tail -1 $O/ncu_full_c4.log
timeout 900 ncu $NCUF -k regex:k_fast -s 25 -c 2 -o $O/prof_fast_neg python bench.py --workload neg --steps 5 --warmup 3 > $O/ncu_full_neg.log 2>&1; tail -1 $O/ncu_full_neg.log
timeout 600 python tools/c5_grid.py 0 96 64 32 > $O/c5_grid.json 2>&1; tail -1 $O/c5_grid.json
bash tools/gpu_c4exp.sh ${1:-extra}_c4x
