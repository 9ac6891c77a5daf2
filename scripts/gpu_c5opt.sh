O=gpurun_out/${TAG:-c5opt}
mkdir -p $O
for cfg in "base:" "split2:SLK_TC_SPLIT=2" "qb1:SLK_TC_QB=1" "qb2:SLK_TC_QB=2" "bc2:SLK_TC_BC=2" "hs1:SLK_TC_HS=1"; do
  name=${cfg%%:*}; env=${cfg#*:}
  env $env SLK_TRACE=1 timeout 300 python bench.py --config C5 --no-cpu-baseline --steps 2 --warmup 2 > $O/c5_$name.log 2>&1
done
