timeout 900 python -m pytest tests/test_gpu_vp.py -q --timeout 300 2>&1 | tail -3
