# RESIDENT schedule: timeline (debug build), parity tests, bench of auto/fused/resident
mkdir -p gpurun_out
ODPO_LIB=build_variants/libodpo_resdbg.so timeout 120 python profiles/res_debug.py > gpurun_out/res_debug.log 2>&1
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or world_size or poison" > gpurun_out/res_tests.log 2>&1; echo rc=$? >> gpurun_out/res_tests.log
for s in auto fused resident; do timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule $s 2>&1 | tail -1 > gpurun_out/res_bench_$s.json; done
