O=gpurun_out/${TAG:-r02z}
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python scripts/sanitize_run.py > $O/sanitizer_racecheck.log 2>&1; echo "rc=$?" >> $O/sanitizer_racecheck.log
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3.log 2>&1
SLK_TRACE=1 timeout 300 python scripts/bench_dendro.py 1000000 > $O/bench_dendro.log 2>&1
