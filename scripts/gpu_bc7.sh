O=gpurun_out/${TAG:-bc7}
mkdir -p $O
for cfg in C3 C2 C5 C1; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 > $O/bench_${cfg}.log 2>&1; done
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 3 > $O/bench_C3_trace.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect "tests/test_configs_gpu.py::test_pipeline_digest[C3]" --deselect "tests/test_configs_gpu.py::test_pipeline_digest[C5]" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
