timeout 900 ncu --set full --clock-control none -k regex:"k_lmhead_fwd2|nvjet" -s 2 -c 2 -o /tmp/lf -f python profiles/r02/lmhead_grad_bench.py llama --quick > /dev/null 2>&1
python profiles/summarize_ncu.py r02x_llama_head llama head "" /tmp/lf.ncu-rep 2>&1 | grep -vE "^$" | head -50
ncu -i /tmp/lf.ncu-rep --page details --csv 2>/dev/null | grep -E "HighPipe|Power|Clock|SM Frequency" | cut -d, -f5,13-16 | head -12
