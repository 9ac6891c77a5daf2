O=gpurun_out/${TAG:-final2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
for cfg in C3 C2 C5 C1; do timeout 600 python bench.py --config $cfg > $O/bench_${cfg}.log 2>&1; done
timeout 600 python bench.py --impl reference --config C3 > $O/bench_reference_C3.log 2>&1
for d in 32 128 512; do timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline > $O/bench_C4_d${d}_k8.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch_run.log 2>&1
timeout 300 python scripts/bench_mst.py > $O/bench_mst.log 2>&1
SLK_TRACE=1 timeout 300 python scripts/bench_dendro.py 1000000 > $O/bench_dendro.log 2>&1
