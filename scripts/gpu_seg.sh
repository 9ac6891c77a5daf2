O=gpurun_out/${TAG:-seg}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --config C5 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C5.log 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C5 --no-cpu-baseline --steps 1 --warmup 1 > $O/bench_C5_trace.log 2>&1
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3.log 2>&1
timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C2.log 2>&1
