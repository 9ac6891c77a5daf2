O=gpurun_out/${TAG:-am}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cfg in C3 C2 C5 C1; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 > $O/bench_${cfg}.log 2>&1; done
for d in 32 128 512; do timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline > $O/bench_C4_d${d}_k8.log 2>&1; done
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/bench_C3_trace.log 2>&1
