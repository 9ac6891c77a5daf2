O=gpurun_out/${TAG:-prof}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
for cfg in C3 C2 C5 C1; do timeout 600 python bench.py --config $cfg > $O/bench_${cfg}.log 2>&1; done
timeout 600 python bench.py --impl reference --config C3 > $O/bench_reference_C3.log 2>&1
for d in 32 128 512; do timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline > $O/bench_C4_d${d}_k8.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch_run.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_bc -c 1 -o $O/bc_cc python scripts/profile_scan.py cc 1000000 64 50 1 > $O/bc_cc.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan -c 1 -o $O/tc_knn python scripts/profile_scan.py knn 1000000 64 50 15 > $O/tc_knn.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:boruvka -c 1 -o $O/boruvka python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $O/boruvka.log 2>&1
