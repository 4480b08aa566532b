# bench.py with CUDA-graph replays of the step (default) vs eager Python calls (--no-graph)
O=gpurun_out/graph_ab; mkdir -p $O
for cfg in tiny pythia rho llama rho_k4; do
  timeout 600 python bench.py --config $cfg --no-cpu --no-e2e > $O/bench_${cfg}_graph.json 2> $O/bench_${cfg}_graph.err
  timeout 600 python bench.py --config $cfg --no-cpu --no-e2e --no-graph > $O/bench_${cfg}_eager.json 2> $O/bench_${cfg}_eager.err
done
timeout 600 python bench.py --config pythia --loss rloo --no-cpu --no-e2e --no-aux > $O/bench_pythia_rloo_graph.json 2> $O/bench_pythia_rloo_graph.err
for f in $O/*.json; do python - "$f" <<'PY'
import json, sys
f = sys.argv[1]
try:
    d = json.loads(open(f).read().strip().splitlines()[-1])
except Exception as e:
    print(f, "ERR", e); sys.exit()
r = d["roofline"]; a = d.get("roofline_factored") or {}
print(f.split("/")[-1], round(d["value"], 1), "step", round(d["ms_per_step"], 4), "loss", round(r["loss_ms_mean"], 4),
      "frac", round(r["frac"], 4), "fact", round(a.get("frac", 0), 4), a.get("loss_ms_mean"),
      d["config"].get("launch", "")[:10], d["config"].get("graph_matches_eager"), d.get("status"))
PY
done
tail -3 $O/*.err
