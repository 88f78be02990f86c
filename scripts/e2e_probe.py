import sys, time; sys.path.insert(0, '/root/repo')
import torch, dataclasses
from paper_1911_07722_b200 import ColumnMatrix, GlmProblem, LabeledDataset, run_syscd
from paper_1911_07722_b200.configs import workload
cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workload(cfg_id)
pb = wl.problem; m = pb.data.matrix
host = torch.empty(m._dev_dense.shape, dtype=torch.float32, pin_memory=True); host.copy_(m._dev_dense)
labels = pb.data.labels.copy()
cfg = dataclasses.replace(wl.solver, metrics_every=10_000_000)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dev = host.to("cuda", non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    mm = ColumnMatrix.from_device(dev, m.n_rows); ds = LabeledDataset(mm, labels, pb.data.orientation)
    p2 = GlmProblem.build(ds, pb.loss, pb.reg.lam, reg=pb.reg.kind); torch.cuda.synchronize(); t2 = time.perf_counter()
    res = run_syscd(p2, cfg); _ = res.alpha.sum(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"h2d {1e3*(t1-t0):.1f} ms ({host.numel()*4/(t1-t0)/1e9:.1f} GB/s)  build {1e3*(t2-t1):.1f}  run {1e3*(t3-t2):.1f}  epochs {sum(mm_.seconds for mm_ in res.metrics)*1e3:.1f}")
    del dev, mm, ds, p2

import os
if os.environ.get("E2E_PROFILE"):
    import cProfile, pstats
    dev = host.to("cuda"); torch.cuda.synchronize()
    pr = cProfile.Profile(); pr.enable()
    mm = ColumnMatrix.from_device(dev, m.n_rows); ds = LabeledDataset(mm, labels, pb.data.orientation)
    p2 = GlmProblem.build(ds, pb.loss, pb.reg.lam, reg=pb.reg.kind)
    res = run_syscd(p2, cfg); _ = res.alpha.sum(); torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumtime").print_stats(40)
