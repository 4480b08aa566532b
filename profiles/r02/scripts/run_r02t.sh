timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_safety.py -q --timeout 300 2>&1 | tail -15
