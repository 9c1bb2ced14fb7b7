python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bupdate -s 25 -c 1 -o gpurun_out/prof_bupdate python tools/exp_c4.py > gpurun_out/ncu_bupd.log 2>&1
tail -1 gpurun_out/ncu_bupd.log
