timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_golden.py -m gpu -q 2>&1 | grep -E "Error|assert |FAILED|passed|failed|^E " | head -30
