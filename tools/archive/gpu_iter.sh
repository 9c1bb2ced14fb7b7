# test + bench + ncu launch list + full capture of update and scan
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 python bench.py --steps 300 --warmup 10 --cpu-budget 2 > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -3 gpurun_out/bench.err
cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_scan|k_probe|k_ingest|k_finalize" -s 100 -c 5 -o gpurun_out/prof_all python bench.py --steps 5 --warmup 3 --skip-cpu --skip-latency > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
