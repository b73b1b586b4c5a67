import cProfile, pstats, sys, time, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2104_10949_b200 as M
import bench
imgs, labels = bench._synthetic(128, 100)
def run(iters):
    cfg = M.TrainConfig(0.01, 128, iters, 0)
    job = (lambda ctx: M.train_private(ctx, M.alexnet_cifar(), cfg, (imgs, labels) if ctx.party == 0 else None))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    M.run_in_process(job, seed=0); torch.cuda.synchronize()
    return time.perf_counter() - t0
run(2)
for it in (1, 2, 4, 12):
    print(it, run(it))
pr = cProfile.Profile(); pr.enable(); run(12); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
