O=gpurun_out/${TAG:-hs2}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cfg in C5 C1 C3 C2; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_$cfg.log 2>&1; done
