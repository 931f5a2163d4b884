#!/bin/bash
# Round profile capture on the GPU box (one GPU).  Summarise here with
# scripts/summarize_ncu.py (traffic / full / launches).
#  1. every launch of one 4096^2 G solve: DRAM bytes, duration, global atom/red and
#     shared atom throughput per kernel.  Grids >= 2^23 px run a round's push launches as
#     a CUDA while-graph, whose kernels ncu does not replay one by one: the per-launch
#     push-kernel captures use option pr_graph=0 (the same launches, driven from the host
#     every 2 launches), and the bench launch list profiles each round graph as one entry
#     (--graph-profiling graph).
#  2. ncu --set full (source level) of the push kernel (an early, dense launch and a
#     mid-solve one), the global-relabel BFS (owner_bfs_kernel) and its preparation pass,
#     the min-cut reach ring and the assignment kernels at n = 4096
#  3. the bench's launch list
mkdir -p gpurun_out
P=${P:-r02}
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum
REPS=1 timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${P}_traffic.csv \
  python scripts/grid_sweep.py 4096 G "pr_graph=0,pr_batch=2" > gpurun_out/${P}_traffic_solve.log 2>&1
F="ncu --set full --import-source on --clock-control none"
REPS=1 timeout 600 $F -k regex:pr_list_kernel -s 0 -c 1 -o gpurun_out/${P}_pr_list_early -f python scripts/grid_trace.py 4096 G trace=0 pr_graph=0 pr_batch=2 > /dev/null 2>&1
REPS=1 timeout 600 $F -k regex:pr_list_kernel -s 40 -c 1 -o gpurun_out/${P}_pr_list_mid -f python scripts/grid_trace.py 4096 G trace=0 pr_graph=0 pr_batch=2 > /dev/null 2>&1
REPS=1 timeout 600 $F -k regex:owner_bfs_kernel -s 3 -c 1 -o gpurun_out/${P}_owner_bfs -f python scripts/grid_trace.py 4096 G trace=0 > /dev/null 2>&1
REPS=1 timeout 600 $F -k regex:relabel_init_kernel -s 3 -c 1 -o gpurun_out/${P}_relabel_init -f python scripts/grid_trace.py 4096 G trace=0 > /dev/null 2>&1
REPS=1 timeout 600 $F --kernel-name-base demangled -k "regex:ring_kernel<.int.1>" -s 0 -c 1 -o gpurun_out/${P}_ring_cut -f python scripts/grid_trace.py 4096 G trace=0 > /dev/null 2>&1
REPS=1 timeout 600 $F -k regex:refine_rounds_kernel -s 2 -c 1 -o gpurun_out/${P}_assign_rounds -f python scripts/assign_one.py 4096 M10000 > /dev/null 2>&1
REPS=1 timeout 600 $F -k regex:price_update_kernel -s 2 -c 1 -o gpurun_out/${P}_assign_pu -f python scripts/assign_one.py 4096 M10000 > /dev/null 2>&1
timeout 900 ncu --graph-profiling graph --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${P}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-virtual-bands > gpurun_out/${P}_bench_ncu.log 2>&1
ls -la gpurun_out
