timeout 600 python -m pytest tests/test_gpu_raster.py -q -x -k "chunked or pinned" 2>&1 | tail -3
