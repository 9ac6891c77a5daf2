O=gpurun_out/${TAG:-pv}
mkdir -p $O
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 2 > $O/bench_C3.log 2>&1
SLK_FORCE_PIVOT=1 SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 2 > $O/bench_C3_pivot.log 2>&1
SLK_FORCE_PIVOT=1 SLK_TC_NPROD=3 SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 2 > $O/bench_C3_pivot_np3.log 2>&1
SLK_FORCE_PIVOT=1 SLK_TRACE=1 timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 2 > $O/bench_C2_pivot.log 2>&1
