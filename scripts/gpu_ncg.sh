O=gpurun_out/${TAG:-ncg}
mkdir -p $O
for v in "" ncg2; do
  SLK_LIB_VARIANT=$v timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3_$v.log 2>&1
  SLK_LIB_VARIANT=$v SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 2 --warmup 2 > $O/bench_C3_trace_$v.log 2>&1
done
SLK_LIB_VARIANT=ncg2 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -m gpu -q -x > $O/pytest_ncg2.log 2>&1; echo rc=$? >> $O/pytest_ncg2.log
