O=gpurun_out/${TAG:-kb}
mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_configs_gpu.py tests/test_acceptance_gpu.py -m gpu -q -x -rf -k "dendrogram or fold or single_linkage or errors or C1 or C2 or C3 or c04 or c01" > $O/pytest_dendro.log 2>&1; echo "rc=$?" >> $O/pytest_dendro.log
SLK_TRACE=1 timeout 300 python scripts/bench_dendro.py 1000000 > $O/bench_dendro.log 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 --warmup 3 > $O/bench_C3_trace.log 2>&1
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3.log 2>&1
