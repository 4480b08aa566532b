#!/bin/bash
# Round-1 factored-gradient record: ncu launch lists + full captures of the unscaled kernel
# (pythia: geometry 0, llama: geometry 1), and the default bench line (scaled + aux unscaled).
mkdir -p gpurun_out
for cfg in pythia llama; do
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01u_${cfg}_launches.csv \
      python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu --no-aux --gradient unscaled > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"k_engine" -s 4 -c 1 \
      -o gpurun_out/r01u_${cfg}_prof -f python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu --no-aux \
      --gradient unscaled > /dev/null 2>&1
done
python bench.py > gpurun_out/r01u_bench_pythia.json 2> gpurun_out/r01u_bench_pythia.err
ls -la gpurun_out | tail -12
