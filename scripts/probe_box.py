# One-off probe of the GPU box: host RAM/cores, H2D/D2H pinned bandwidth.
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().split("\n")[:3]
out["cpu"] = [l for l in open("/proc/cpuinfo").read().split("\n") if l.startswith("model name")][:1]
out["smi"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
for size_mb in (32, 92, 256, 1024):
    n = size_mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
    s.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = max(3, 2048 // size_mb)
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    e1.synchronize()
    h2d = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(reps):
            h.copy_(d, non_blocking=True)
        e1.record(s)
    e1.synchronize()
    d2h = n * reps / (e0.elapsed_time(e1) * 1e-3) / 1e9
    out[f"h2d_{size_mb}MB_GBs"] = round(h2d, 2)
    out[f"d2h_{size_mb}MB_GBs"] = round(d2h, 2)
# pinned alloc cost for 8 GB
t = time.time(); big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True); out["pin_8GB_s"] = round(time.time() - t, 2)
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
