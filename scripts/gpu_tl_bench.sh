O=gpurun_out/${TAG:-tl}
mkdir -p $O
rm -f $O/*.tl
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/knn.tl timeout 300 python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/cc.tl timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc.log 2>&1
for f in $O/*.tl; do echo $f; python scripts/timeline.py $f; done > $O/summary.txt 2>&1
SLK_TRACE=1 timeout 300 python bench.py --config C3 --no-cpu-baseline > $O/bench_C3.log 2>&1
timeout 300 python bench.py --config C5 --no-cpu-baseline > $O/bench_C5.log 2>&1
