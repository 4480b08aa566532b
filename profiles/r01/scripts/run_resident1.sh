mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "resident" > gpurun_out/res_tests.log 2>&1; echo rc=$? >> gpurun_out/res_tests.log
for s in auto fused resident; do timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule $s 2>&1 | tail -1 > gpurun_out/res_bench_$s.json; done
