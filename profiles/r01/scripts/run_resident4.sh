# RESIDENT (TMEM stash + L2-backed rows): parity, timeline, cap sweep
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or world_size or poison or inplace or full_size" > gpurun_out/res_tests.log 2>&1; echo rc=$? >> gpurun_out/res_tests.log
ODPO_LIB=build_variants/libodpo_resdbg.so timeout 120 python profiles/res_debug.py > gpurun_out/res_debug.log 2>&1
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule fused 2>&1 | tail -1 > gpurun_out/res_bench_fused.json
for c in 0 1 2 3 4 6; do timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule resident --lookahead $c 2>&1 | tail -1 > gpurun_out/res_bench_cap$c.json; done
