timeout 600 python -m pytest tests/test_codec.py tests/test_control.py -q 2>&1 | tail -3
