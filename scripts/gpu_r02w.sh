O=gpurun_out/${TAG:-w}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cfg in C3 C5 C2; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 > $O/bench_${cfg}.log 2>&1; done
timeout 300 python scripts/bench_mst.py > $O/bench_mst.log 2>&1
