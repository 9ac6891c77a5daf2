# ncu --set full of the k-NN and cross-colour scan launches at C3 scale
O=gpurun_out/${TAG:-ncu}
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan -c 1 -o $O/knn python scripts/profile_scan.py knn 1000000 64 50 15 > $O/knn.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_scan -c 1 -o $O/cc python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc.log 2>&1
