O=gpurun_out/${TAG:-mst}
mkdir -p $O
timeout 300 python scripts/bench_mst.py > $O/bench_mst.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_acceptance_gpu.py tests/test_cli_gpu.py -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 > $O/bench_C3.log 2>&1
