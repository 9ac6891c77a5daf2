O=gpurun_out/${TAG:-bc2}
mkdir -p $O
rm -f $O/*.tl
for bc in 1 0; do
  SLK_TC_BC=$bc SLK_TRACE=1 timeout 300 python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn_bc$bc.log 2>&1
  SLK_TC_BC=$bc SLK_TRACE=1 timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc_bc$bc.log 2>&1
done
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/knn.tl timeout 300 python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn_tl.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TIMELINE=$O/cc.tl timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc_tl.log 2>&1
for f in $O/*.tl; do echo $f; python scripts/timeline.py $f; done > $O/summary.txt 2>&1
