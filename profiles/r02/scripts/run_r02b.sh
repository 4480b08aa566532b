# round 2: regime tests after the fp32 (x - m) k2 fix and the all -inf batch guard
timeout 600 python -m pytest tests/test_gpu_regimes.py -q --timeout 300 -x -k "V4133 and flat and fused" 2>&1 | tail -60 > gpurun_out/r02b_first.log
timeout 900 python -m pytest tests/test_gpu_regimes.py -q --timeout 300 2>&1 | grep -v "^$" | tail -60 > gpurun_out/r02b_regimes.log
tail -3 gpurun_out/r02b_regimes.log
