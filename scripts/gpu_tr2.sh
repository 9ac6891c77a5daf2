O=gpurun_out/${TAG:-tr2}
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -rf > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 2 --warmup 1 > $O/bench_tr2.log 2>&1; echo "rc=$?" >> $O/bench_tr2.log
