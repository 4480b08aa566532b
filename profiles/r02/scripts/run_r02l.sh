# Last record after the NEXT-2 dynamic tile order: smoke, the default bench line, Pythia line
O=gpurun_out/r02l; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_llama.json 2> $O/bench_llama.err
timeout 900 python bench.py --config pythia > $O/bench_pythia.json 2> $O/bench_pythia.err
for f in $O/bench_*.json; do python - "$f" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r = d["roofline"]; a = d.get("aux_lmhead_pythia") or {}
print(sys.argv[1], round(d["value"], 1), round(r["loss_ms_mean"], 3), round(r["frac"], 4), r["traffic"], d["clocks"]["sm_mhz"],
      {k: round(a[k], 3) for k in ("ms", "step_chunked_ms", "step_unfused_ms", "grad_ms") if k in a}, d["config"]["graph_matches_eager"])
PY
done
