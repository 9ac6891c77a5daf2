O=gpurun_out/${TAG:-krt}
mkdir -p $O
timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -rf -k "dendrogram or fold or single_linkage or errors" > $O/pytest_dendro.log 2>&1; echo "rc=$?" >> $O/pytest_dendro.log
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3.log 2>&1
SLK_HOST_FOLD=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3_hostfold.log 2>&1
timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 6 --warmup 3 > $O/bench_C3_b.log 2>&1
