O=gpurun_out/${TAG:-bc4}
mkdir -p $O
rm -f $O/*.tl
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 2 > $O/bench_C3.log 2>&1
SLK_TC_BC=0 SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline --steps 2 > $O/bench_C3_old.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/knn.tl timeout 300 python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn_tl.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/cc.tl timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc_tl.log 2>&1
for f in $O/*.tl; do echo $f; python scripts/timeline.py $f; done > $O/summary.txt 2>&1
for cfg in C5 C2; do SLK_TRACE=1 timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 2 > $O/bench_${cfg}.log 2>&1; SLK_TC_BC=0 SLK_TRACE=1 timeout 300 python bench.py --config $cfg --no-cpu-baseline --steps 2 > $O/bench_${cfg}_old.log 2>&1; done
