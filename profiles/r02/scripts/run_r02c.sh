# round 2: full GPU suite + smoke after the parity/safety changes
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -x 2>&1 | tail -40 > gpurun_out/r02c_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1
tail -3 gpurun_out/r02c_gpu.log; tail -2 gpurun_out/r02c_smoke.log
