O=gpurun_out/${TAG:-bc6}
mkdir -p $O
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 > $O/bench_C3.log 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 3 > $O/bench_C3_trace.log 2>&1
timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 3 > $O/bench_C2.log 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 1 --warmup 3 > $O/bench_C2_trace.log 2>&1
