# round 2 measurement: default bench (LLaMA), the other configs, ncu launch list + --set full
# captures of the dominant kernel (scaled and factored) per config
mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
lscpu > $O/lscpu.txt 2>&1
timeout 900 python bench.py > $O/bench_llama.json 2> $O/bench_llama.err
for cfg in pythia rho tiny rho_k4; do
  timeout 600 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_llama.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
for cfg in llama pythia rho; do
  for g in scaled unscaled; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_engine" -s 4 -c 1 \
      -o $O/full_${cfg}_${g} -f python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu \
      --no-aux --gradient $g > /dev/null 2>&1
  done
done
ls -la $O
cat $O/bench_llama.json | head -c 3000
