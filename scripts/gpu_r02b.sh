set -x
O=gpurun_out/r02b
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q -rA --durations=40 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_C3.log 2>&1
timeout 300 python bench.py --config C1 > $O/bench_C1.log 2>&1
timeout 300 python bench.py --config C2 > $O/bench_C2.log 2>&1
timeout 300 python bench.py --config C5 > $O/bench_C5.log 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_run.py > $O/sanitizer_$tool.log 2>&1; echo "rc=$?" >> $O/sanitizer_$tool.log
done
