# bench lines (no cpu/e2e) for WLS under each VARIANTS entry (A=B[,C=D] or base)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > gpurun_out/pytest_gpu.log; grep -q failed gpurun_out/pytest_gpu.log && echo "!!!!!!!! PYTEST FAILED !!!!!!!!"
: > gpurun_out/bench_var.jsonl
for v in ${VARIANTS:-base}; do
  for w in ${WLS:-cfg2 cfg3}; do
    env $(echo $v | tr ',' ' ' | sed 's/^base$//') timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e | sed "s/^/$v /" >> gpurun_out/bench_var.jsonl 2>> gpurun_out/bench_var.err
  done
done
cat gpurun_out/pytest_gpu.log
python - <<'PY'
import json
for l in open("gpurun_out/bench_var.jsonl"):
    v, j = l.split(" ", 1)
    d = json.loads(j)
    print(v, d["config"]["workload"], "ms %.4f" % d["ms_per_step"], "Gelem/s %.2f" % d["value"], "fwd %.4f (%.3f)" % (d["fwd_ms"], d["fwd_frac"]),
          "bwd %.4f (%.3f)" % (d.get("bwd_ms", 0), d.get("bwd_frac", 0)))
PY
