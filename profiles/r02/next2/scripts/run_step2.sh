mkdir -p gpurun_out
python -m pytest tests/test_lmhead.py -q -x -m gpu 2>&1 | tail -3
for i in 1 2; do python profiles/r02/lmhead_grad_bench.py --quick; done
ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/step_breakdown2.csv python profiles/r02/next2/scripts/step_breakdown.py > gpurun_out/step_breakdown2.log 2>&1
python - <<'PY'
import csv,io
txt=open("gpurun_out/step_breakdown2.csv").read().splitlines()
i=next(k for k,l in enumerate(txt) if l.startswith('"ID"'))
rows=list(csv.DictReader(io.StringIO("\n".join(txt[i:]))))
by={}
for r in rows:
    by.setdefault(int(r["ID"]),{})[r["Metric Name"]]=(r["Kernel Name"],r["Metric Value"])
for i in sorted(by)[-42:-9]:
    m=by[i]; k=m["gpu__time_duration.sum"][0][:60]
    print(i,k,float(m["gpu__time_duration.sum"][1])/1e3,round(float(m["sm__cycles_elapsed.avg.per_second"][1])/1e6))
PY
