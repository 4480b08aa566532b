O=gpurun_out/r02g; mkdir -p $O
timeout 300 python profiles/r02/debug_grad.py 2>&1 | tail -20
timeout 900 python -m pytest tests/test_lmhead.py tests/test_gpu_safety.py -q -x --timeout 600 2>&1 | tail -3
timeout 600 python profiles/r02/lmhead_grad_bench.py > $O/grad_pythia.json 2>&1; cat $O/grad_pythia.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lmh" --csv --log-file $O/grad_launches.csv python profiles/r02/lmhead_grad_bench.py --quick > /dev/null 2>&1
python profiles/summarize_ncu.py r02g_grad pythia grad $O/grad_launches.csv > /dev/null 2>&1; cp profiles/r02/ncu/r02g_grad_ncu_summary.md $O/ 2>/dev/null; cat $O/r02g_grad_ncu_summary.md
