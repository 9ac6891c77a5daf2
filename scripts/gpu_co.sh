O=gpurun_out/${TAG:-co}
mkdir -p $O
for d in 512 128 32; do
  timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline --steps 2 --warmup 1 > $O/c4_d${d}.log 2>&1
  SLK_NO_COMMON_ORDER=1 timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline --steps 2 --warmup 1 > $O/c4_d${d}_noco.log 2>&1
done
timeout 900 python -m pytest tests/test_configs_gpu.py tests/test_parity_gpu.py -m gpu -q -x -k "c4 or large_d or knn" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
