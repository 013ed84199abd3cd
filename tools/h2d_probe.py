"""Host->device bandwidth probe on the GPU box (pinned buffers like bench.py's e2e leg)."""
import os, subprocess, time, torch
print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout)
dev = torch.device("cuda", 0)
for gb in (1, 8):
    n = gb * 2**30 // 4
    t0 = time.perf_counter()
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    t_pin = time.perf_counter() - t0
    d = torch.empty(64 * 2**20 // 4, dtype=torch.float32, device=dev)
    res = []
    for rep in range(6):
        torch.cuda.synchronize()
        t = time.perf_counter()
        for off in range(0, min(n, 32 * len(d)), len(d)):
            d.copy_(h[off:off + len(d)], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        res.append(round(min(n, 32 * len(d)) * 4 / dt / 1e9, 1))
    print(f"{gb} GB pinned (pin {t_pin:.1f}s): H2D GB/s over 2 GB windows: {res}", flush=True)
    del h
