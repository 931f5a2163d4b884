#!/bin/bash
# assignment tuning sweep on the GPU box: price-update threshold (relabels)
for pu in ${PUS:-64 128 256 1024}; do
  echo "PU=$pu"; FM_PU_THRESHOLD=$pu timeout 300 python scripts/bench_assign.py ${N:-4096} pu 2>&1 | tail -3
done
