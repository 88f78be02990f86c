"""Config-4 sparse epoch cost split: logistic-dual (Newton) vs svm-dual
(closed form) on the same CSC matrix, several partition counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_07722_b200 import SolverConfig, run_syscd
from paper_1911_07722_b200.configs import device_problem
from paper_1911_07722_b200.objective import GlmProblem, SmoothLoss

scale = float(os.environ.get("SCALE", "1.0"))
pb = device_problem(4, scale, 0)
hinge = GlmProblem.build(pb.data, SmoothLoss.hinge(), 1e-6)
for P in [int(p) for p in os.environ.get("PS", "512").split(",")]:
    for name, prob in (("logistic", pb), ("hinge", hinge)):
        cfg = SolverConfig(K=1, P=P, bucket_size=64, T1=3, seed=0)
        torch.cuda.synchronize()
        res = run_syscd(prob, cfg)
        print(f"P={P} {name}: epoch ms {[round(m.seconds * 1e3, 2) for m in res.metrics[1:]]}"
              f" obj {[round(m.objective, 6) for m in res.metrics[1:]]}", flush=True)
