#!/bin/bash
# A/B of the push kernel: v2 (pr_tile_kernel) vs v3 (pr_list_kernel) and v3 passes per visit
S=${S:-4096}
for K in G S; do
  echo "== $K v2"; FM_PR_KERNEL=0 timeout 120 python scripts/tune_grid.py $S $K 0:0 2>&1 | tail -1 | cut -c1-400
  for kl in ${KLS:-32 64 128}; do
    echo "== $K v3 k=$kl"; FM_PR_KERNEL=1 FM_K_LOCAL_LIST=$kl timeout 120 python scripts/tune_grid.py $S $K 0:0 2>&1 | tail -1 | cut -c1-400
  done
done
