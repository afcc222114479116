timeout 600 python -m pytest tests/test_gpu_raster.py tests/test_golden.py tests/test_dropin.py -x -q 2>&1 | tail -2
timeout 600 python tools/ab_variants.py run raster c2 5
