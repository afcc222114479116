timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/prof_workload.py raster c5 2
timeout 600 python tools/prof_workload.py raster c2 5
