# round 2: (1) tcgen05 backward GEMM + new tests, (2) factored A/B: round-1 lib vs now (BREV on /
# off), (3) bench lines, (4) ncu launch list + --set full, summarised ON the box (reports are
# too big to bring back)
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests/test_lmhead.py tests/test_gpu_safety.py -q --timeout 600 -x 2>&1 | tail -30 > $O/tests_lmhead_safety.log
tail -3 $O/tests_lmhead_safety.log
ab() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']; print('$1', d['config']['workload'], 'loss_ms %.3f frac %.3f' % (r['loss_ms_mean'], r['frac']), d['clocks'])"; }
for cfg in llama pythia; do
  (cd build_variants/r01 && timeout 300 python bench.py --config $cfg --gradient unscaled --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu 2>/dev/null | ab r01) >> $O/ab_unscaled.log 2>&1
  timeout 300 python bench.py --config $cfg --gradient unscaled --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu 2>/dev/null | ab now_brev1 >> $O/ab_unscaled.log 2>&1
  timeout 300 python bench.py --config $cfg --gradient unscaled --steps 20 --warmup 5 --no-aux --no-e2e --no-cpu --lib build_variants/libodpo_brev0.so 2>/dev/null | ab now_brev0 >> $O/ab_unscaled.log 2>&1
done
cat $O/ab_unscaled.log
timeout 900 python bench.py > $O/bench_llama.json 2> $O/bench_llama.err
for cfg in pythia rho tiny rho_k4; do
  timeout 600 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_llama.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
mkdir -p /tmp/ncu
for cfg in llama pythia rho; do
  for g in scaled unscaled; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_engine" -s 4 -c 1 \
      -o /tmp/ncu/full_${cfg}_${g} -f python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu \
      --no-aux --gradient $g > /dev/null 2>&1
    L=""; [ $cfg = llama ] && [ $g = scaled ] && L=$O/launches_llama.csv
    python profiles/summarize_ncu.py r02e_${cfg}_${g} $cfg $g $L /tmp/ncu/full_${cfg}_${g}.ncu-rep > /dev/null 2>&1
  done
done
cp -r profiles/r02/ncu $O/ncu
cp /tmp/ncu/full_llama_scaled.ncu-rep $O/ 2>/dev/null
du -sh $O; ls $O $O/ncu
