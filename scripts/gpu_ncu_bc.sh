O=gpurun_out/${TAG:-ncubc}
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_bc -c 1 -o $O/cc python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc.log 2>&1
