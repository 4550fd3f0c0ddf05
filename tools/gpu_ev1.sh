# Round-2 evidence: GPU tests, a strict 1,500-case stress sweep and the three
# compute-sanitizer tools over tools/sanitize.py (writes gpurun_out/r02_*).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02_gputests.txt 2>&1; tail -2 gpurun_out/r02_gputests.txt
timeout 1500 python tools/stress_random.py 1500 23 > gpurun_out/r2_stress_random3.txt 2>&1; tail -2 gpurun_out/r2_stress_random3.txt
rm -f gpurun_out/r02_sanitizers.txt
for t in memcheck racecheck synccheck; do
  echo "== $t" >> gpurun_out/r02_sanitizers.txt
  timeout 900 compute-sanitizer --tool $t --print-limit 20 $( [ $t = synccheck ] && echo --num-cuda-barriers 8192 ) python tools/sanitize.py 2>&1 | tail -6 >> gpurun_out/r02_sanitizers.txt
done
tail -20 gpurun_out/r02_sanitizers.txt
