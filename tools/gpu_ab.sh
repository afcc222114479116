timeout 900 python -m pytest tests/test_gpu_raster.py tests/test_gpu_fullsize.py tests/test_dropin.py -q -x 2>&1 | tail -2
