O=gpurun_out/r02i; mkdir -p $O
timeout 600 python profiles/r02/lmhead_grad_bench.py --quick 2>&1 | tail -1
for v in gemmg8 gemmkb gemmkb_g8; do
  timeout 600 python -c "
import sys; sys.argv=['x','--quick']
import paper_2410_18252_b200 as odpo; odpo.LIB_PATH='build_variants/libodpo_$v.so'
exec(compile(open('profiles/r02/lmhead_grad_bench.py').read(), 'profiles/r02/lmhead_grad_bench.py', 'exec'), {'__name__': '__main__', '__file__': 'profiles/r02/lmhead_grad_bench.py'})
" 2>&1 | tail -1 | sed "s/^/$v /"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file $O/grad_launches.csv python profiles/r02/lmhead_grad_bench.py --quick > /dev/null 2>&1
python profiles/summarize_ncu.py r02i_grad pythia grad $O/grad_launches.csv > /dev/null 2>&1; cp profiles/r02/ncu/r02i_grad_ncu_summary.md $O/ 2>/dev/null; cat $O/r02i_grad_ncu_summary.md
