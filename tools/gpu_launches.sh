# usage: bash tools/gpu_launches.sh <workload> <tag>: per-launch device times of our kernels
W=${1:-cfg2}; TAG=${2:-launches}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:scan2d -c 12 --csv \
  --log-file gpurun_out/${TAG}_${W}.csv python bench.py --workload $W --steps 3 --warmup 3 --no-e2e --no-cpu --no-accurate > /dev/null 2>&1
