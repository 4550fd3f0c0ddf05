# GPU: parity tests (quick) + shape timings, optionally under several env settings
#   SHAPES="S,H,W,N ..."  VARIANTS="ENV=1 ENV=2 ..." (each variant: space-free A=B[,C=D])
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
: > gpurun_out/shapes.jsonl
for v in ${VARIANTS:-base}; do
  echo "## $v" >> gpurun_out/shapes.jsonl
  env $(echo $v | tr ',' ' ' | sed 's/^base$//') timeout 600 python tools/time_shapes.py ${SHAPES:-128,200,200,16 1664,200,16,16} >> gpurun_out/shapes.jsonl 2>&1
done
cat gpurun_out/pytest_gpu.log gpurun_out/shapes.jsonl | cut -c1-160
