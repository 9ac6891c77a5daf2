O=gpurun_out/${TAG:-ld2}
mkdir -p $O
SLK_TC_BC=2 SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/c3_bc2.log 2>&1
SLK_LIB_VARIANT=ld2 SLK_TC_BC=2 SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/c3_bc2_ld2.log 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/c3_base.log 2>&1
