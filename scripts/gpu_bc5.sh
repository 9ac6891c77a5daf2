O=gpurun_out/${TAG:-bc5}
mkdir -p $O
for cfg in C3 C5 C2 C1; do
  timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 > $O/bench_${cfg}.log 2>&1
  SLK_TC_BC=0 timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 3 > $O/bench_${cfg}_old.log 2>&1
done
