O=gpurun_out/${TAG:-dbg}
mkdir -p $O
SLK_DEBUG_CERT=1 SLK_TRACE=1 timeout 300 python bench.py --config C5 --no-cpu-baseline --steps 1 --warmup 1 > $O/bench_C5.log 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 1 > $O/bench_C3.log 2>&1
