# Headline spread (three back-to-back default bench runs) and the multi-rank bench path (two
# ranks sharing the GPU over gloo, with and without the peer-memory stats exchange)
O=gpurun_out/r02j; mkdir -p $O
for i in 1 2 3; do timeout 900 python bench.py > $O/bench_llama_$i.json 2> $O/bench_llama_$i.err; done
export ODPO_SHARE_GPU=1 ODPO_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --config pythia --steps 5 --warmup 3 --no-aux --no-e2e --stats-exchange > $O/two_ranks_exchange.json 2> $O/two_ranks_exchange.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 2 --config pythia --steps 5 --warmup 3 --no-aux --no-e2e > $O/two_ranks_allreduce.json 2> $O/two_ranks_allreduce.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > $O/two_ranks_reference.json 2> $O/two_ranks_reference.err
for f in $O/*.json; do echo $f; tail -1 $f | cut -c1-400; done
