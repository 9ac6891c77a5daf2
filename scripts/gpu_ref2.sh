O=gpurun_out/${TAG:-ref2}
mkdir -p $O
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/bench_C3_trace.log 2>&1
