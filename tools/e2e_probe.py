"""Where does end-to-end (pinned host input) time go? Run on a GPU box."""
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2011_03910_b200 as p
from paper_2011_03910_b200 import synth

dev = torch.device("cuda", 0)
gen = synth.make("cfg1", device=dev, seed=0)
B, N = 32, 9
batches = [gen.next_batch(B) for _ in range(N)]
host = [p.HeadOutputs(tuple(h.cpu().pin_memory() for h in b.heads),
                      tuple(e.cpu().contiguous(memory_format=torch.channels_last).pin_memory() for e in b.embs))
        for b in batches]
torch.cuda.synchronize()
# 1. raw H2D bandwidth from the pinned tensors
x = host[0].heads[2]
y = torch.empty_like(x, device=dev)
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter(); 
for _ in range(10): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 10
print(f"H2D {x.numel()*4/1e6:.1f} MB: {x.numel()*4/dt/1e9:.1f} GB/s", flush=True)
for pipe in (True, False):
    cap = p.Capacity(streams=1, max_frames=B, max_candidates=512, max_detections=256, max_tracks=256)
    bt = p.BatchTracker(1, frames_per_update=B, capacity=cap, pipeline=pipe)
    hout = bt.host_output(B)
    bt.update(host[0], host_out=hout)
    lib = bt.engine.lib
    lib.tf_set_profiling(bt.engine.ctx, 1)
    walls = []
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(1, N):
        a = time.perf_counter()
        bt.update(host[i], host_out=hout, sync=False)
        walls.append((time.perf_counter() - a) * 1e3)
    bt.join(); torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3
    import ctypes as C
    f, s_, n = C.c_double(), C.c_double(), C.c_int64()
    lib.tf_kernel_times(bt.engine.ctx, C.byref(f), C.byref(s_), C.byref(n))
    print(f"pipeline={pipe}: total {tot:.2f} ms for {N-1} steps = {(N-1)*B/tot*1e3:.0f} frames/s; host ms per update call "
          f"{[round(w, 2) for w in walls]}; frame kernel {f.value/max(n.value,1):.3f} ms, assoc {s_.value/max(n.value,1):.3f} ms", flush=True)
    # device-resident for comparison
    bt3 = p.BatchTracker(1, frames_per_update=B, capacity=cap, pipeline=pipe)
    bt3.update(batches[0]); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(1, N): bt3.update(batches[i], sync=False)
    bt3.join(); torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3
    print(f"  device-resident wall: {(N-1)*B/tot*1e3:.0f} frames/s", flush=True)
