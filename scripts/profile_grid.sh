#!/bin/bash
# On the GPU box: per-round trace at 4096^2, ncu source-level capture of pr_tile_kernel
# and bfs_tile_kernel mid-solve, and the bench launch list.
mkdir -p gpurun_out
S=${S:-4096}
FM_TRACE=1 timeout 120 python scripts/tune_grid.py $S G 0:0 > gpurun_out/trace_$S.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pr_tile_kernel -s ${SKIP:-40} -c 2 \
  -o gpurun_out/prof_pr_tile -f python scripts/tune_grid.py $S G 0:0 > gpurun_out/ncu_pr.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfs_tile_kernel -s 60 -c 2 \
  -o gpurun_out/prof_bfs_tile -f python scripts/tune_grid.py $S G 0:0 > gpurun_out/ncu_bfs.log 2>&1
if [ -n "$LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
fi
ls -la gpurun_out
