# A/B of the scan variants on one box: parity suite, then C3/C5/C2 bench under each setting
O=gpurun_out/${TAG:-ab}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -x --deselect "tests/test_configs_gpu.py::test_pipeline_digest[C3]" --deselect "tests/test_configs_gpu.py::test_pipeline_digest[C5]" > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cfg in C3 C5 C2; do
  SLK_TRACE=1 timeout 300 python bench.py --config $cfg --no-cpu-baseline > $O/bench_${cfg}.log 2>&1
  SLK_TC_NPROD=3 timeout 300 python bench.py --config $cfg --no-cpu-baseline > $O/bench_${cfg}_np3.log 2>&1
done
