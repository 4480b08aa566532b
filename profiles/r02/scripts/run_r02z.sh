timeout 2400 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unscaled.py -q --timeout 600 -k "resident or psync" --odpo-lib build_variants/libodpo_experimental.so 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
