O=gpurun_out/${TAG:-c4}
mkdir -p $O
for d in 32 128; do
  SLK_TC_BC=2 SLK_TRACE=1 timeout 600 python bench.py --config C4 --d $d --k 8 --no-cpu-baseline --steps 2 --warmup 1 > $O/c4_d${d}_bc2.log 2>&1
done
SLK_TC_NPROD=1 SLK_TRACE=1 timeout 900 python bench.py --config C4 --d 512 --k 8 --no-cpu-baseline --steps 1 --warmup 1 > $O/c4_d512_np1.log 2>&1
