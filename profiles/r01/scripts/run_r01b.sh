# Round-1 (second session) evidence: full GPU suite, default bench, ncu of the lmhead kernel and
# of the RESIDENT kernel, lmhead raster sweep
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01b_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r01b_gpu_tests.log
timeout 300 python bench.py > gpurun_out/r01b_bench_pythia.json 2> gpurun_out/r01b_bench_pythia.err
: > gpurun_out/lmh_bench.log
for g in 64 128 256; do echo G=$g >> gpurun_out/lmh_bench.log; ODPO_LMH_G=$g timeout 300 python profiles/lmhead_bench.py >> gpurun_out/lmh_bench.log 2>&1; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lmhead_fwd -s 3 -c 1 -o gpurun_out/r01b_lmhead -f python profiles/lmhead_bench.py > gpurun_out/r01b_lmhead_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:k_resident -s 2 -c 1 -o gpurun_out/r01b_resident -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-aux --schedule resident --lookahead 0 > gpurun_out/r01b_resident_ncu.log 2>&1
ls gpurun_out
