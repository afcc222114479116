timeout 900 python -m pytest tests/test_gpu_voxel.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -2
