O=gpurun_out/${TAG:-tl}
mkdir -p $O
rm -f $O/*.tl
for np in 1 3; do
SLK_LIB_VARIANT=timeline SLK_TC_NPROD=$np SLK_TIMELINE=$O/knn_np$np.tl timeout 300 python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn_np$np.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TC_NPROD=$np SLK_TIMELINE=$O/cc_np$np.tl timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc_np$np.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TC_QB=1 SLK_TC_NPROD=$np SLK_TIMELINE=$O/cc1_np$np.tl timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc1_np$np.log 2>&1
done
for f in $O/*.tl; do echo $f; python scripts/timeline.py $f; done > $O/summary.txt 2>&1
