# scratch A/B run (edited per experiment; see tools/ab_variants.py)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/ab_variants.py run raster c2 5
timeout 600 python tools/ab_variants.py run raster c5 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python tools/prof_workload.py raster c2 1 > /dev/null 2>&1
