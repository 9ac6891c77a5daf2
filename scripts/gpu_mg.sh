O=gpurun_out/${TAG:-mg}
mkdir -p $O
timeout 900 python -m pytest tests/test_multigpu_gpu.py -m gpu -q -rf > $O/pytest_mg.log 2>&1; echo "rc=$?" >> $O/pytest_mg.log
python - > $O/mg_timing.log 2>&1 <<'PY'
import time, numpy as np, torch
import paper_2306_16354_b200 as slk
from paper_2306_16354_b200.synthetic import bench_points
x = bench_points(1_000_000, 64, 50, seed=0)
cfg = slk.LinkageConfig(n_clusters=50, k=15, seed=0)
for g in [1, 2, 4]:
    for rep in range(3):
        t = time.perf_counter(); r = slk.single_linkage_result(x, cfg, n_gpus=g); dt = time.perf_counter() - t
    print("n_gpus", g, "s", round(dt, 4), "iters", r.connect_iters, r.timings)
PY
