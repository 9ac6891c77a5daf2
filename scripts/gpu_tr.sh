O=gpurun_out/${TAG:-tr}
mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 1 > $O/bench_tr2.log 2>&1; echo "rc=$?" >> $O/bench_tr2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --steps 2 --warmup 1 --impl reference > $O/bench_tr2_ref.log 2>&1; echo "rc=$?" >> $O/bench_tr2_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --config C4 --d 32 --k 8 > $O/bench_tr2_c4.log 2>&1; echo "rc=$?" >> $O/bench_tr2_c4.log
