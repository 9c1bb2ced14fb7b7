# f4 GPU parity + device-search hang probe (diagnostic round)
O=gpurun_out/${1:-f4b}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -20 $O/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_f4.py -q -p no:cacheprovider > $O/f4.log 2>&1; tail -30 $O/f4.log
timeout 1500 python tools/hang_probe.py --rounds 400 --limit 15 > $O/hang.log 2>&1; echo "probe rc=$?"; tail -12 $O/hang.log
