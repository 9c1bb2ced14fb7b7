# Support-row pitch experiment: C3b with the paper's Alg. 3
# scans (use_gather = 0), 5 fresh processes per build, pitch pad 0 / 16 / 144 words.
# Usage: gpurun --timeout 1800 -- 'bash tools/gpu_pitch.sh'
O=gpurun_out/pitch; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for pad in 16 144; do
  python -c "from paper_2507_18413_b200 import build as b; b.build(out='/tmp/libct_pad$pad.so', extra=['-DCT_SUP_PITCH_PAD=$pad'])" >> $O/build.log 2>&1
done
CT_LIB_PATH=/tmp/libct_pad144.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > $O/pytest_pad144.log 2>&1; tail -1 $O/pytest_pad144.log
for r in 1 2 3 4 5; do
  for pad in 0 16 144; do
    if [ $pad = 0 ]; then L=""; else L="CT_LIB_PATH=/tmp/libct_pad$pad.so"; fi
    env $L timeout 300 python bench.py --workload c3b --no-gather --steps 200 --warmup 10 --skip-cpu > $O/c3b_pad${pad}_$r.json 2> $O/c3b_pad${pad}_$r.err
    [ $r = 1 ] && env $L timeout 300 python bench.py --workload c3b --steps 200 --warmup 10 --skip-cpu > $O/c3bg_pad${pad}_$r.json 2> $O/c3bg_pad${pad}_$r.err
  done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/pitch/*.json')):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); print(f, round(d['value']), round(d['ms_per_step'] * 1e3, 1))
    except Exception as e:
        print(f, 'ERR', e)
PY
