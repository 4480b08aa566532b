O=gpurun_out/r02n; mkdir -p $O
./profiles/r02/racecheck_probe/probe
compute-sanitizer --tool racecheck --print-limit 5 ./profiles/r02/racecheck_probe/probe > $O/probe_racecheck.log 2>&1
grep -E "Race reported|ERROR SUMMARY|probe done" $O/probe_racecheck.log | head -8
compute-sanitizer --tool memcheck ./profiles/r02/racecheck_probe/probe 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none -k regex:"k_gemm" -c 2 -o /tmp/g -f python profiles/r02/lmhead_grad_bench.py --quick > /dev/null 2>&1
python profiles/summarize_ncu.py r02n_gemm pythia gemm "" /tmp/g.ncu-rep 2>&1 | grep -vE "^$" | head -40
ncu -i /tmp/g.ncu-rep --page details --csv 2>/dev/null | grep -E "HighPipe|Stall|Warp Cycles|Issue Slots|Tensor" | cut -d, -f5,12-16 | head -20
