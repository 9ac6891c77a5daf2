O=gpurun_out/${TAG:-c2bc}
mkdir -p $O
for bc in 1 2; do SLK_TC_BC=$bc SLK_TRACE=1 timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 2 --warmup 2 > $O/c2_bc$bc.log 2>&1; done
for bc in 1 2; do SLK_TC_BC=$bc timeout 600 python bench.py --config C2 --no-cpu-baseline --steps 5 --warmup 3 > $O/c2n_bc$bc.log 2>&1; done
