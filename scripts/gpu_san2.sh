O=gpurun_out/${TAG:-san2}
mkdir -p $O
timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python scripts/sanitize_run.py > $O/sanitizer_racecheck.log 2>&1; echo "rc=$?" >> $O/sanitizer_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 50 python scripts/sanitize_run.py > $O/sanitizer_synccheck.log 2>&1; echo "rc=$?" >> $O/sanitizer_synccheck.log
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cfg in C3 C2; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 > $O/bench_${cfg}.log 2>&1; done
