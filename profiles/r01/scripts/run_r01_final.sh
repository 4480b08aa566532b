#!/bin/bash
# Round-1 record: bench lines for every config + ncu launch list + full capture of the fused kernel.
mkdir -p gpurun_out
python bench.py > gpurun_out/r01_bench_pythia.json 2> gpurun_out/r01_bench_pythia.err
for c in tiny rho llama; do
  timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e > gpurun_out/r01_bench_$c.json 2> gpurun_out/r01_bench_$c.err
done
timeout 600 python bench.py --config strong --steps 1 --warmup 1 > gpurun_out/r01_bench_strong.json 2> gpurun_out/r01_bench_strong.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r01_bench_reference.json 2> gpurun_out/r01_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_final_launches.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_engine" -s 4 -c 2 \
    -o gpurun_out/r01_final_prof -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out | tail -20
