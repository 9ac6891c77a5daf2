O=gpurun_out/${TAG:-kp}
mkdir -p $O
for kp in 8 4; do SLK_TC_KP1=$kp SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 1 --warmup 2 > $O/bench_C3_kp$kp.log 2>&1; done
for kp in 8 4; do SLK_TC_KP1=$kp timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 3 > $O/bench_C3_kp${kp}_nt.log 2>&1; done
