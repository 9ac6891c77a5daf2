O=gpurun_out/${TAG:-vo}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 --warmup 3 > $O/bench_C3_trace.log 2>&1
for cfg in C3 C2 C5; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_${cfg}.log 2>&1; done
SLK_FLAT_GATHER=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3_gather.log 2>&1
timeout 600 python bench.py --config C4 --d 128 --k 8 --no-cpu-baseline > $O/bench_C4_d128.log 2>&1
