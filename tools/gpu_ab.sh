timeout 900 python -m pytest tests/test_gpu_raster.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
timeout 600 python tools/ab_variants.py run raster c5 2
timeout 600 python tools/ab_variants.py run raster c5 2
timeout 600 python tools/ab_variants.py run raster c2 3
