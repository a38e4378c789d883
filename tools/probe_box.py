"""One-off probe of the GPU box: host cores/RAM, GPU, pinned H2D/D2H and D2D bandwidth."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["sched_affinity"] = len(os.sched_getaffinity(0))
with open("/proc/meminfo") as f:
    out["meminfo"] = [l.strip() for l in f.readlines()[:3]]
out["lscpu"] = subprocess.run("lscpu | head -20", shell=True, capture_output=True, text=True).stdout
out["smi"] = subprocess.run("nvidia-smi; nvidia-smi topo -m", shell=True, capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
n = 4 << 30
t0 = time.time()
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
out["pin_4GiB_s"] = time.time() - t0
d = torch.empty(n, dtype=torch.uint8, device=dev)
d2 = torch.empty(n, dtype=torch.uint8, device=dev)
def timeit(fn, reps=5):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize(); s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize(); best = min(best, s.elapsed_time(e) / 1e3)
    return best
out["h2d_GBps"] = n / timeit(lambda: d.copy_(h, non_blocking=True)) / 1e9
out["d2h_GBps"] = n / timeit(lambda: h.copy_(d, non_blocking=True)) / 1e9
out["d2d_GBps_rw"] = 2 * n / timeit(lambda: d2.copy_(d)) / 1e9
free, total = torch.cuda.mem_get_info()
out["mem_free_total"] = [free, total]
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
