# parity tests + short bench lines (no cpu/e2e) for the given workloads
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
: > gpurun_out/bench_wls.jsonl
for w in ${WLS:-cfg2 cfg3}; do
  env $VARS timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e >> gpurun_out/bench_wls.jsonl 2>> gpurun_out/bench_wls.err
done
tail -3 gpurun_out/pytest_gpu.log
python - <<'PY'
import json
for l in open("gpurun_out/bench_wls.jsonl"):
    d = json.loads(l)
    print(d["config"]["workload"], "ms %.4f" % d["ms_per_step"], "Gelem/s %.2f" % d["value"], "fwd %.4f (%.3f)" % (d["fwd_ms"], d["fwd_frac"]),
          "bwd %.4f (%.3f)" % (d.get("bwd_ms", 0), d.get("bwd_frac", 0)), d["plan"])
PY
