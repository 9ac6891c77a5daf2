O=gpurun_out/${TAG:-kb2}
mkdir -p $O
SLK_TRACE=1 timeout 300 python scripts/bench_dendro.py 1000000 > $O/bench_dendro.log 2>&1
SLK_KRT_GRID_ONLY=1 SLK_TRACE=1 timeout 300 python scripts/bench_dendro.py 1000000 > $O/bench_dendro_grid.log 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 --warmup 3 > $O/bench_C3_trace.log 2>&1
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3.log 2>&1
SLK_KRT_GRID_ONLY=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3_grid.log 2>&1
