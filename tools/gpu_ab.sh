# scratch A/B run (edited per experiment; see tools/ab_variants.py)
timeout 600 python tools/ab_variants.py run raster c2 5
timeout 600 python tools/ab_variants.py run raster c5 1
