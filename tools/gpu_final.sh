#!/bin/bash
# End-of-round evidence pass (writes gpurun_out/r02_*): GPU tests, a bench line
# per workload, Table 3, the reference-API path, the reference arm, ncu launch
# lists and the cfg2 full captures.  (Sanitizers: tools/gpu_ev1.sh.)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests.txt 2>&1; tail -2 gpurun_out/r02_gputests.txt
for w in cfg2 cfg1 cfg2m cfg3 cfg4a cfg4b cfg4c cfg4d cfg5; do
  timeout 900 python bench.py --workload $w > gpurun_out/r02_bench_$w.json 2> gpurun_out/r02_bench_$w.err
  echo "$w: $(head -c 300 gpurun_out/r02_bench_$w.json | cut -c 100-260)"
done
timeout 600 python bench.py --workload cfg2m --bc-reduce fixed --no-cpu --no-e2e --no-accurate > gpurun_out/r02_bench_cfg2m_fixed.json 2>&1
timeout 600 python bench.py --compare > gpurun_out/r02_table3.json 2>&1
timeout 900 python bench.py --api shim --steps 3 > gpurun_out/r02_shim.json 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_reference_cfg2.json 2>&1
for w in cfg1 cfg2 cfg2m cfg3 cfg4a cfg4b cfg4c cfg4d cfg5; do bash tools/gpu_launches.sh $w r02_launches; done
bash tools/gpu_prof.sh cfg2 scan2d_bwd_tile2 r02_bwd
bash tools/gpu_prof.sh cfg2 scan2d_fwd_tile2 r02_fwd
for k in bwd fwd; do
  python tools/ncu_details.py gpurun_out/r02_${k}_cfg2.ncu-rep > gpurun_out/r02_cfg2_${k}_full.txt 2>&1
  rm -f gpurun_out/r02_${k}_cfg2.ncu-rep
done
