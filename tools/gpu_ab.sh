timeout 600 python tools/e2e_phase.py
timeout 600 python tools/prof_workload.py raster c2 5
