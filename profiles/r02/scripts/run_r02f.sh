# round 2: NEXT-4 exchange tests, NEXT-2 backward timing + launch list
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_vp.py -q --timeout 600 2>&1 | tail -30 > $O/tests_vp.log
tail -3 $O/tests_vp.log
timeout 600 python profiles/r02/lmhead_grad_bench.py > $O/grad_pythia.json 2>&1
cat $O/grad_pythia.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"lmh|transpose" --csv --log-file $O/grad_launches.csv python -c "
import sys; sys.argv=['x']
exec(open('profiles/r02/lmhead_grad_bench.py').read().replace('for ch in (None, 4736, 9472, 18944, 27136):', 'for ch in (None,):'))
" > /dev/null 2>&1
python profiles/summarize_ncu.py r02f_grad pythia grad $O/grad_launches.csv > $O/grad_launches.md 2>&1; cp profiles/r02/ncu/r02f_grad_ncu_summary.md $O/ 2>/dev/null
head -30 $O/r02f_grad_ncu_summary.md
