"""H2D bandwidth of a pinned buffer, before and after binding the process to
the GPU's NUMA-local CPUs (pynvml)."""
import os, time
import torch

def h2d(nbytes=3_200_000_000):
    host = torch.empty(nbytes // 4, dtype=torch.float32, pin_memory=True)
    host.fill_(1.0)
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        dev = host.to("cuda", non_blocking=True); torch.cuda.synchronize()
        best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
        del dev
    return best

torch.cuda.init()
print("cpus", len(os.sched_getaffinity(0)), "h2d GB/s", round(h2d(), 1))
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    n = os.cpu_count()
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
    cpus = [64 * w + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1]
    os.sched_setaffinity(0, cpus)
    print("gpu-local cpus", len(cpus), "h2d GB/s", round(h2d(), 1))
except Exception as e:
    print("affinity failed:", e)
