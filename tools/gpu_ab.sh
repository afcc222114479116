timeout 600 python tools/bitcmp_raster.py
timeout 600 python tools/ab_variants.py run raster c2 5
timeout 600 python tools/ab_variants.py run raster c2 5
