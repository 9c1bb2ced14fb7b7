#!/bin/bash
# GPU test pass on a gpurun box: build, then pytest -m gpu (args forwarded).
# Usage: gpurun -- 'bash tools/gpu_tests.sh TAG [pytest args...]'
TAG=${1:-run}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
nproc > $OUT/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo build failed; tail -30 $OUT/build.log; exit 1; }
timeout 3300 python -m pytest tests -m gpu -q -rf -p no:cacheprovider "$@" > $OUT/pytest.log 2>&1
rc=$?
echo "pytest rc=$rc" >> $OUT/pytest.log
tail -40 $OUT/pytest.log
exit $rc
