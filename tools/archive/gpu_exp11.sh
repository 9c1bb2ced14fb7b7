python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pipelined or config3_bulk" 2>&1 | tail -1
for mode in zc dma zc dma; do
  if [ $mode = dma ]; then export CT_HOST_DMA=1; else unset CT_HOST_DMA; fi
  timeout 300 python bench.py --workload c3bulk --steps 400 --warmup 10 --skip-cpu --skip-latency 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$mode', round(d['value']), round(e['value']), round(e['host_enqueue_us_per_step'],1), round(e['sync_call']['value']))"
done
