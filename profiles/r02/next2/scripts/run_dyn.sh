# Dynamic tile order of the CTA-pair head kernels: parity (tests/test_lmhead.py), DRAM per
# LLaMA-head forward (ncu metrics), sustained clock/time, the chunked step vs unfused
O=gpurun_out/${TAG:-dyn}; mkdir -p $O
timeout 600 python -m pytest tests/test_lmhead.py -q -x --timeout 300 2>&1 | tail -3 > $O/lmhead_tests.log
cat $O/lmhead_tests.log
timeout 300 python profiles/r02/next2/scripts/head_once.py > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:"k_lmhead_fwd2|nvjet" -s 2 -c 2 --csv python profiles/r02/next2/scripts/head_once.py 2>/dev/null | grep -v "^==" > $O/ncu_head.csv
timeout 300 python profiles/r02/next2/scripts/power_probe.py 2>&1 | tail -4 | sed 's/^{/{"lib": "dyn", /' > $O/probe.jsonl
timeout 300 python profiles/r02/next2/scripts/power_probe.py build_variants/libodpo_lmhstatic.so 2>&1 | tail -4 | sed 's/^{/{"lib": "static", /' >> $O/probe.jsonl
cat $O/probe.jsonl
timeout 600 python profiles/r02/lmhead_grad_bench.py llama --quick > $O/grad_llama.json 2>&1
timeout 600 python profiles/r02/lmhead_grad_bench.py --quick > $O/grad_pythia.json 2>&1
cat $O/grad_llama.json; cat $O/grad_pythia.json
