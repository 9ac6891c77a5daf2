O=gpurun_out/${TAG:-ncuref}
mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:refine_kernel -c 2 -o $O/refine python scripts/profile_scan.py cc 1000000 64 50 1 > $O/refine_cc.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:refine_kernel -c 1 -o $O/refine_knn python scripts/profile_scan.py knn 1000000 64 50 15 > $O/refine_knn.log 2>&1
