timeout 300 ncu --set full --import-source on --clock-control none -k regex:bfs_ring_kernel -s 4 -c 1 -o gpurun_out/prof_ring -f python scripts/tune_grid.py 4096 G 0:0 > gpurun_out/ncu_r.log 2>&1
