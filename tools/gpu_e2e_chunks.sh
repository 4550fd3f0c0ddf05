# e2e (host operands through scan2d_train_host) vs chunk count, per workload
mkdir -p gpurun_out
: > gpurun_out/e2e_chunks.txt
for w in ${WLS:-cfg2 cfg3}; do
  for c in ${CHUNKS:-0 8 16 32}; do
    timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu --e2e-chunks $c 2>>gpurun_out/e2e_chunks.err |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', 'chunks $c', 'e2e', d['e2e']['value'], d['e2e']['unit'], 'dev', round(d['value'],2))" >> gpurun_out/e2e_chunks.txt
  done
done
cat gpurun_out/e2e_chunks.txt
