O=gpurun_out/${TAG:-pf}
mkdir -p $O
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_C3.log 2>&1
timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 5 --warmup 3 > $O/bench_C2.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
