# RESIDENT: exp2 split and forward-warp variants (cap 2)
mkdir -p gpurun_out
for pv in 0 1 2 3 4 5 6; do timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule resident --exp2-split $pv 2>&1 | tail -1 > gpurun_out/res_bench_pv$pv.json; done
for pv in 0 2 4; do ODPO_LIB=build_variants/libodpo_fw8.so timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule resident --exp2-split $pv 2>&1 | tail -1 > gpurun_out/res_bench_fw8pv$pv.json; done
for pv in 0 2 4; do timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-aux --schedule fused --exp2-split $pv 2>&1 | tail -1 > gpurun_out/res_bench_fusedpv$pv.json; done
