# Round-1 end evidence (second session): full GPU suite, smoke, bench lines for every config,
# the reference arm, and the ncu launch list of the default bench
mkdir -p gpurun_out/r01_end
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r01_end/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r01_end/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01_end/smoke.log 2>&1; echo rc=$? >> gpurun_out/r01_end/smoke.log
timeout 300 python bench.py > gpurun_out/r01_end/bench_pythia.json 2> gpurun_out/r01_end/bench_pythia.err
for c in tiny rho llama rho_k4; do timeout 400 python bench.py --config $c --no-cpu > gpurun_out/r01_end/bench_$c.json 2> gpurun_out/r01_end/bench_$c.err; done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r01_end/bench_reference.json 2> gpurun_out/r01_end/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_end/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/r01_end/launches_bench.log 2>&1
ls gpurun_out/r01_end
