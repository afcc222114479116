timeout 600 python tools/ab_variants.py run voxel c3 5
