# round 2, first GPU call: the new logit-regime parity tests against the round-1 kernels
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests/test_gpu_regimes.py -q --timeout 600 2>&1 | tail -80 > gpurun_out/r02a_regimes.log
tail -5 gpurun_out/r02a_regimes.log
