timeout 600 python tools/ab_variants.py run e2e c2 3
timeout 600 python tools/ab_variants.py run e2e c2 3
