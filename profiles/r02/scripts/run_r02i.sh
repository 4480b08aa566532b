#!/bin/bash
# Round-2 measurement record: ncu evidence first (so the bench lines carry roofline.traffic from
# captures on these very sources), then the GPU suite, smoke, every bench line, the reference
# arm, App B losses, NEXT-2 / NEXT-4 side measurements.  ncu reports are summarised on the box.
TAG=${1:-r02i}
O=gpurun_out/$TAG; mkdir -p $O /tmp/ncu
lscpu > $O/lscpu.txt 2>&1; nvidia-smi > $O/nvidia_smi.txt 2>&1
# (1) ncu --set full of the dominant kernel per config and gradient form
for cfg in llama pythia rho tiny rho_k4; do
  for g in scaled unscaled; do
    # scaled: the AUTO (two-pass) call's forward, pair reduction and backward kernels; factored:
    # the row engine's one kernel (the first four k_engine launches are the reference pass)
    if [ $g = scaled ]; then K='regex:k_engine|k_pair_reduce|k_row_bwd'; C=3; else K='regex:k_engine'; C=1; fi
    timeout 900 ncu --set full --clock-control none --import-source on -k $K -s 4 -c $C \
      -o /tmp/ncu/full_${cfg}_${g} -f python bench.py --config $cfg --steps 1 --warmup 3 --no-e2e --no-cpu \
      --no-aux --gradient $g > /dev/null 2>&1
    python profiles/summarize_ncu.py ${TAG}_${cfg}_${g} $cfg $g "" /tmp/ncu/full_${cfg}_${g}.ncu-rep > /dev/null 2>&1
  done
done
# (2) launch list of the default bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_llama.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python profiles/summarize_ncu.py ${TAG}_launches llama scaled_launchlist $O/launches_llama.csv > /dev/null 2>&1
rm -f profiles/r02/ncu/traffic_llama_scaled_launchlist.json
cp -r profiles/r02/ncu $O/ncu
# (3) tests + smoke
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 2>&1 | tail -15 > $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
tail -2 $O/gpu_tests.log; tail -1 $O/smoke.log
# (4) bench lines
timeout 1200 python bench.py > $O/bench_llama.json 2> $O/bench_llama.err
for cfg in pythia rho tiny rho_k4; do
  timeout 900 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err
done
timeout 900 python bench.py --config strong --steps 5 --warmup 3 > $O/bench_strong.json 2> $O/bench_strong.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for cfg in pythia rho llama; do
  for loss in rloo copg prox_rloo sft; do
    timeout 300 python bench.py --config $cfg --loss $loss --no-aux --no-e2e --no-cpu 2>/dev/null | tail -1 >> $O/bench_losses.jsonl
  done
done
# (5) NEXT-2 (LLaMA head) and NEXT-4 (per-rank shard kernels, gathered vs in-kernel exchange)
timeout 900 python profiles/r02/lmhead_grad_bench.py llama --quick > $O/grad_llama.json 2>&1
timeout 600 python profiles/r02/lmhead_grad_bench.py --quick > $O/grad_pythia.json 2>&1
for cfg in pythia rho llama; do for W in 2 8; do
  timeout 300 python profiles/vp_bench.py --config $cfg --W $W >> $O/vp_per_rank.jsonl 2>&1
  timeout 300 python profiles/vp_bench.py --config $cfg --W $W --put >> $O/vp_per_rank.jsonl 2>&1
done; done
ls -la $O | head -50
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/*/bench_*.json")):
    pass
PY
