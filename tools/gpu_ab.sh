timeout 900 python -m pytest tests/test_gpu_raster.py -q -x 2>&1 | tail -2
timeout 600 python tools/prof_workload.py e2e c2 3
