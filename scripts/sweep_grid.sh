#!/bin/bash
# grid tuning sweep on the GPU box: relabel budget divisor x k_local
S=${S:-4096}; K=${K:-G}
for rd in ${RDS:-1 4 16}; do
  echo "RELABEL_DIV=$rd"; FM_RELABEL_DIV=$rd timeout 300 python scripts/tune_grid.py $S $K ${CFGS:-16:0 32:0 64:0} 2>&1 | tail -3
done
