#!/bin/bash
# One compute-sanitizer tool per gpurun call (never several in one call), on
# the small all-kernels workload, after the same workload exited 0 plainly.
#   bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
T=${1:?tool}
O=gpurun_out/san; mkdir -p $O
timeout 600 python tools/sanitize_small.py > $O/plain_$T.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 2400 compute-sanitizer --tool $T --print-limit 200 --log-file $O/$T.log \
  python tools/sanitize_small.py > $O/$T.out 2>&1
echo "sanitizer_rc=$?" >> $O/$T.out
tail -3 $O/$T.log
