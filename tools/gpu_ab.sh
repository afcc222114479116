# scratch A/B run (edited per experiment; see tools/ab_variants.py)
timeout 600 python tools/ab_variants.py run voxel c3 3
