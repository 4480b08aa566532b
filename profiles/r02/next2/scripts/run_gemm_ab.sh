# Backward GEMMs of the chunked step: raster group (ODPO_GEMM_G) and dynamic order for all calls
O=gpurun_out/gemm_ab; mkdir -p $O
for i in 1 2; do
for L in main build_variants/libodpo_gg4.so build_variants/libodpo_gg8.so build_variants/libodpo_gg32.so build_variants/libodpo_dyn0.so build_variants/libodpo_dyn0gg8.so; do
  X=""; [ $L != main ] && X=$L
  timeout 600 python profiles/r02/lmhead_grad_bench.py llama --quick $X 2>&1 | tail -1 | sed "s#^{#{\"lib\": \"$L\", #" >> $O/llama.jsonl
  timeout 300 python profiles/r02/lmhead_grad_bench.py --quick $X 2>&1 | tail -1 | sed "s#^{#{\"lib\": \"$L\", #" >> $O/pythia.jsonl
done; done
python - <<'PY'
import json
for f in ["gpurun_out/gemm_ab/llama.jsonl", "gpurun_out/gemm_ab/pythia.jsonl"]:
    for l in open(f):
        try:
            d = json.loads(l)
        except Exception:
            print(l[:200]); continue
        print(f.split("/")[-1], d["lib"].split("/")[-1], "fwd %.2f grad %.2f chunked %.2f unfused %.2f" % (d["fwd_ms"], d["grad_ms_chunk_None"], d["step_chunked_ms"], d["step_unfused_ms"]))
PY
