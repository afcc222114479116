# scratch driver for one-off GPU A/B runs (edited per experiment; see tools/ab_variants.py)
timeout 600 python tools/ab_variants.py run raster c2 5
