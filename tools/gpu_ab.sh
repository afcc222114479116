timeout 600 python tools/ab_variants.py run raster c5 2
timeout 600 python tools/ab_variants.py run raster c5 2
