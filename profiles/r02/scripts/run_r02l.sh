timeout 600 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "psync" --odpo-lib build_variants/libodpo_experimental.so 2>&1 | tail -5
timeout 300 python -m pytest tests/test_gpu_parity.py -q --timeout 120 -k "psync" 2>&1 | tail -2
