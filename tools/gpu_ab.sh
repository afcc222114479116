timeout 600 python tools/ab_variants.py run voxel c3 5
timeout 600 python tools/ab_variants.py run raster c2 5
