#!/bin/bash
# A/B on the GPU box: default build vs 4-CTA/SM build, op steps 1/2/4/8
for lib in ${LIBS:-paper_1110_6231_b200/libfm_b200.so}; do
  for st in 1 2 4 8; do
    echo "LIB=$lib STEPS=$st"
    FM_LIB_PATH=$lib FM_OP_STEPS=$st timeout 100 python scripts/tune_grid.py ${S:-4096} ${K:-G} 0:0 2>&1 | tail -1 | cut -c1-330
  done
done
