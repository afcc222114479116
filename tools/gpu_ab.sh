timeout 600 python -m pytest tests/test_gpu_raster.py -q -x -k "pinned" 2>&1 | tail -2
