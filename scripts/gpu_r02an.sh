O=gpurun_out/${TAG:-an}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for d in 512; do timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline > $O/bench_C4_d${d}_k8.log 2>&1; done
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 > $O/bench_C3.log 2>&1
