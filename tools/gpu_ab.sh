timeout 600 python -m pytest tests/test_gpu_raster.py -q -x 2>&1 | tail -2
timeout 600 python tools/ab_variants.py run e2e c2 3
timeout 600 python tools/ab_variants.py run e2e c2 3
