timeout 600 python -m pytest tests/test_gpu.py -q -k "random_configs" 2>&1 | tail -15
