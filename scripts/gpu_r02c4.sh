O=gpurun_out/${TAG:-r02c4}
mkdir -p $O
timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -k "tied" -rf > $O/pytest_tied.log 2>&1; echo "rc=$?" >> $O/pytest_tied.log
for d in 32 128 512; do timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline > $O/bench_C4_d${d}_k8.log 2>&1; done
