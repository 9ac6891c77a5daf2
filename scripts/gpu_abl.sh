O=gpurun_out/${TAG:-abl}
mkdir -p $O
for v in base nomma noconv noepi; do
  if [ $v = base ]; then L=""; else L=$v; fi
  SLK_LIB_VARIANT=$L SLK_TRACE=1 timeout 300 python scripts/profile_scan.py cc 1000000 64 50 1 > $O/cc_$v.log 2>&1
done
