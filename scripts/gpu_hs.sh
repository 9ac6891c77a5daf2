O=gpurun_out/${TAG:-hs}
mkdir -p $O
for hs in 2 4; do
  SLK_BC_HS=$hs timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 > $O/bench_C3_hs$hs.log 2>&1
  SLK_BC_HS=$hs SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/trace_C3_hs$hs.log 2>&1
  SLK_BC_HS=$hs SLK_TC_BC=2 SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/trace_C3_bc2_hs$hs.log 2>&1
  SLK_BC_HS=$hs timeout 300 python bench.py --config C2 --no-cpu-baseline --steps 3 > $O/bench_C2_hs$hs.log 2>&1
done
SLK_BC_HS=4 timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_multigpu_gpu.py tests/test_configs_gpu.py -m gpu -q -x > $O/pytest_hs4.log 2>&1; echo "rc=$?" >> $O/pytest_hs4.log
SLK_BC_HS=4 SLK_TC_BC=2 timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_acceptance_gpu.py -m gpu -q -x > $O/pytest_hs4_bc2.log 2>&1; echo "rc=$?" >> $O/pytest_hs4_bc2.log
