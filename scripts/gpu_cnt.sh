O=gpurun_out/${TAG:-cnt}
mkdir -p $O
SLK_LIB_VARIANT=timeline SLK_TIMELINE=/tmp/knn.tl SLK_TRACE=1 timeout 300 python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn.log 2>&1
SLK_LIB_VARIANT=timeline SLK_TIMELINE=/tmp/knn.tl SLK_TRACE=1 timeout 300 python scripts/profile_scan.py knn 100000 128 50 15 > $O/knn_c2.log 2>&1
