timeout 300 python -m pytest tests/test_grid_gpu.py tests/test_bands_gpu.py -x -q 2>&1 | tail -2
for ds in 0 1; do for rd in 2 4 8 16; do echo "== devstop=$ds rd=$rd"; FM_DEVICE_STOP=$ds FM_RELABEL_DIV=$rd timeout 60 python scripts/tune_grid.py 4096 G 0:0 2>&1 | tail -1 | cut -c1-300;
FM_DEVICE_STOP=$ds FM_RELABEL_DIV=$rd timeout 60 python scripts/tune_grid.py 2048 S 0:0 2>&1 | tail -1 | cut -c1-200; done; done
