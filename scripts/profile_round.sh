#!/bin/bash
# Round profile capture on the GPU box (one GPU): per-kernel DRAM traffic of every
# launch of one 4096^2 solve, full-set captures of the main kernels, and the bench
# launch list.  Summarise here with scripts/summarize_ncu.py.
mkdir -p gpurun_out
REPS=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"pr_list_kernel|bfs_ring_kernel|cut_bits_kernel|bfs_init_bits_kernel|bfs_finalize_tiles_kernel|cut_init_bits_kernel" \
  --csv --log-file gpurun_out/traffic.csv python scripts/tune_grid.py 4096 G 0:0 > gpurun_out/traffic_solve.log 2>&1
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:pr_list_kernel -s 20 -c 2 \
  -o gpurun_out/prof_pr_list -f python scripts/tune_grid.py 4096 G 0:0 > /dev/null 2>&1
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:bfs_ring_kernel -s 2 -c 1 \
  -o gpurun_out/prof_bfs_ring -f python scripts/tune_grid.py 4096 G 0:0 > /dev/null 2>&1
REPS=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:cut_bits_kernel -s 0 -c 2 \
  -o gpurun_out/prof_cut_bits -f python scripts/tune_grid.py 4096 G 0:0 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu.log 2>&1
ls -la gpurun_out
