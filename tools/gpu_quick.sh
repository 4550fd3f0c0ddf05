# quick GPU check: parity tests + cfg2/cfg5 bench lines + launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
for w in ${WL:-cfg2 cfg5}; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
bash tools/gpu_launches.sh cfg2
cat gpurun_out/pytest_gpu.log
