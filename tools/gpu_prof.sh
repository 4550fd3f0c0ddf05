# usage: bash tools/gpu_prof.sh <workload> <kernel-regex> <tag>   (one ncu --set full capture)
W=${1:-cfg2}; K=${2:-scan2d_bwd}; TAG=${3:-prof}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -f -k regex:$K -s 2 -c 1 \
  -o gpurun_out/${TAG}_${W} python bench.py --workload $W --steps 1 --warmup 3 --no-e2e --no-cpu --no-accurate > gpurun_out/${TAG}_${W}.log 2>&1
