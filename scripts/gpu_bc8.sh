O=gpurun_out/${TAG:-bc8}
mkdir -p $O
rm -f $O/*.tl
for cfg in C3 C2 C5; do timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 > $O/bench_${cfg}.log 2>&1; done
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 3 > $O/bench_C3_trace.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/cc.tl timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc_tl.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/knn.tl timeout 300 python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn_tl.log 2>&1
for f in $O/*.tl; do echo $f; python scripts/timeline.py $f; done > $O/summary.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --deselect "tests/test_configs_gpu.py::test_pipeline_digest[C3]" --deselect "tests/test_configs_gpu.py::test_pipeline_digest[C5]" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
