# Final bench record with graph-replayed steps: every config line, the default (driver) line
# twice, the reference arm, the two-rank path, and the launch list of the default command
O=gpurun_out/r02k; mkdir -p $O
timeout 900 python bench.py > $O/bench_llama.json 2> $O/bench_llama.err
timeout 900 python bench.py > $O/bench_llama_2.json 2> $O/bench_llama_2.err
for cfg in pythia rho tiny rho_k4; do timeout 900 python bench.py --config $cfg > $O/bench_$cfg.json 2> $O/bench_$cfg.err; done
timeout 900 python bench.py --config strong --steps 5 --warmup 3 > $O/bench_strong.json 2> $O/bench_strong.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for cfg in pythia rho llama; do
  for loss in rloo copg prox_rloo sft; do
    timeout 300 python bench.py --config $cfg --loss $loss --no-aux --no-e2e --no-cpu 2>/dev/null | tail -1 >> $O/bench_losses.jsonl
  done
done
export ODPO_SHARE_GPU=1 ODPO_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 2 --config pythia --steps 5 --warmup 3 --no-aux --no-e2e > $O/two_ranks.json 2> $O/two_ranks.err
unset ODPO_SHARE_GPU ODPO_DIST_BACKEND
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu > $O/plain_for_ncu.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_llama.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
python profiles/summarize_ncu.py r02k_launches llama scaled_launchlist $O/launches_llama.csv > /dev/null 2>&1
cp profiles/r02/ncu/r02k_launches_ncu_summary.md $O/ 2>/dev/null
rm -f profiles/r02/ncu/traffic_llama_scaled_launchlist.json
ls $O
