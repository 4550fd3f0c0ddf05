# Full GPU evidence pass: parity tests, smoke, bench lines, ncu launch lists + full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
for w in ${WLS:-cfg3 cfg5 cfg1}; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
for w in cfg2 ${WLS:-cfg3 cfg5 cfg1}; do bash tools/gpu_launches.sh $w; done
bash tools/gpu_prof.sh cfg2 scan2d_fwd full_fwd
bash tools/gpu_prof.sh cfg2 scan2d_bwd full_bwd
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; cat gpurun_out/bench_*.json | cut -c1-400
