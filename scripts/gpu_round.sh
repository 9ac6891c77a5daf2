set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_c3.log 2>&1
timeout 300 python bench.py --config C2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1
timeout 300 python bench.py --config C5 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_scan -c 1 -o gpurun_out/tc_scan_full python scripts/profile_scan.py knn 1000000 64 50 15 > gpurun_out/ncu_full.log 2>&1
