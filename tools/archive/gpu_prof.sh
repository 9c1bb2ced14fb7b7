set -x
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fast -s 10 -c 2 -o gpurun_out/prof_fast_c3 python tools/prof_kernels.py c3 14 > gpurun_out/ncu_fast.log 2>&1
tail -n 2 gpurun_out/ncu_fast.log
