timeout 600 python -m pytest tests/test_lmhead.py -q -x --timeout 600 -k "step" 2>&1 | tail -2
timeout 600 python profiles/r02/lmhead_grad_bench.py --quick 2>&1 | tail -1
timeout 1200 python profiles/r02/lmhead_grad_bench.py llama --quick 2>&1 | tail -1
