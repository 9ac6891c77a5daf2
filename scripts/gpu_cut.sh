O=gpurun_out/${TAG:-cut}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for r in a b; do timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 12 --warmup 3 > $O/bench_C3_$r.log 2>&1; done
timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 12 --warmup 3 > $O/bench_C2.log 2>&1
timeout 300 python bench.py --config C5 --no-cpu-baseline --steps 12 --warmup 3 > $O/bench_C5.log 2>&1
