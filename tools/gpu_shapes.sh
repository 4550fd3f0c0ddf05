# GPU: parity tests (quick) + shape timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 python tools/time_shapes.py ${SHAPES:-128,200,200,16 1664,200,16,16 128,200,208,16} > gpurun_out/shapes.jsonl 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/shapes.jsonl
