O=gpurun_out/${TAG:-y}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=10 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py > $O/bench_C3.log 2>&1
