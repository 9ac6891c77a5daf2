O=gpurun_out/${TAG:-v2}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 12 --warmup 3 > $O/bench_C3.log 2>&1
SLK_HOST_FOLD=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 12 --warmup 3 > $O/bench_C3_hostfold.log 2>&1
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 12 --warmup 3 > $O/bench_C3_b.log 2>&1
