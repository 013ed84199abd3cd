"""Benchmark: tracked frames/sec (decode + NMS + association) on B200 vs the CPU reference.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1] [--impl ours|reference]

A *step* is one ``update(head_outputs)`` of the hot path over one batch: for
config 1 (the BASELINE metric's config: 1088x608 heads, 50 objects, single
stream) that is B = 32 consecutive frames of one stream. Every rank runs its
own stream (weak scaling, no data-path collective); only the final per-rank
metrics are gathered with NCCL. Inputs are synthetic head tensors of the named
shape (paper_2011_03910_b200/synth.py), pre-generated on the device; every
step's inputs (32 x 29 MB) exceed the 126 MB L2, so no flush is needed.

* ``value``   device-resident throughput: CUDA events around K steps on the
              launching stream, barrier + synchronize on both sides, max over ranks.
* ``e2e``     the same metric through the C-ABI with pinned HOST inputs and host
              outputs: confidence planes copied H2D, candidate deltas and
              embeddings read in place over PCIe, records copied D2H, all inside
              the timed region.
* ``roofline`` dominant kernel (associate_kernel at config 1), algorithmic bytes
              per launch / its CUDA-event duration, against MEASURED_PEAKS.json.
* ``cpu_baseline`` the CPU oracle port of the reference path (decode oracle +
              Tracker.step restatement, OPENBLAS_NUM_THREADS=1) on a bounded
              sample of the same stream, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

METRIC = "tracked frames/sec (decode+NMS+association) at 1/2/4/8 B200 vs CPU ref"
N_CELLS = 34 * 19 + 68 * 38 + 136 * 76          # 13,566
CONF_BYTES = 8 * 4 * N_CELLS                    # 434,112 B/frame: the 8 conf planes per cell set


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:
            self.N = None

    def _run(self):
        N = self.N
        names = {getattr(N, k, None): k for k in (
            "nvmlClocksThrottleReasonHwSlowdown", "nvmlClocksThrottleReasonHwThermalSlowdown",
            "nvmlClocksThrottleReasonSwThermalSlowdown", "nvmlClocksThrottleReasonSwPowerCap")}
        label = {"nvmlClocksThrottleReasonHwSlowdown": "hw_slowdown",
                 "nvmlClocksThrottleReasonHwThermalSlowdown": "hw_thermal_slowdown",
                 "nvmlClocksThrottleReasonSwThermalSlowdown": "sw_thermal_slowdown",
                 "nvmlClocksThrottleReasonSwPowerCap": "sw_power_cap"}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, k in names.items():
                    if bit and r & bit:
                        self.reasons.add(label[k])
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.N:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.N:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


# ---------------------------------------------------------------------------- reference arm
def cpu_reference_fps(frames_np, seconds_budget=None):
    """Decode oracle + oracle Tracker.step over host frames, sequential (one stream)."""
    from oracle import heads as oh
    from oracle import tracker as ot

    trk = ot.OracleTracker(ot.Settings())
    t0 = time.perf_counter()
    n = 0
    for i, (heads, embs) in enumerate(frames_np):
        _, rows = oh.decode_frame(heads, embs)
        trk.step(i, ot.rows_to_dets(rows, 512))
        n += 1
        if seconds_budget and time.perf_counter() - t0 > seconds_budget:
            break
    return n / (time.perf_counter() - t0), n


def host_frame_iter(batches, limit):
    """Yield (heads, embs) numpy frames from device batches, one frame at a time."""
    n = 0
    for out in batches:
        F = out.frames
        for b in range(F):
            if n >= limit:
                return
            heads = [h[b].cpu().numpy() for h in out.heads]
            embs = [e[b].cpu().numpy() for e in out.embs]
            yield heads, embs
            n += 1


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    import torch

    from paper_2011_03910_b200 import synth

    # identical workload to our arm; generated on the CPU (no GPU work on this arm)
    gen = synth.make(args.config, device="cpu", seed=args.seed)
    B = args.batch
    cores = 1          # single-stream configs: frames of a stream are order-dependent
    sample_frames = B * min(args.steps, 4)
    per_step = []
    from oracle import heads as oh
    from oracle import tracker as ot

    trk = ot.OracleTracker(ot.Settings())
    fidx = 0
    total_frames, total_s = 0, 0.0
    for step in range(args.warmup + args.steps):
        out = gen.next_batch(B)
        frames = [([h[b].numpy() for h in out.heads], [e[b].numpy() for e in out.embs]) for b in range(B)]
        n = B if step >= args.warmup else min(B, 4)      # warm-up steps: a few frames
        t0 = time.perf_counter()
        for heads, embs in frames[:n]:
            _, rows = oh.decode_frame(heads, embs)
            trk.step(fidx, ot.rows_to_dets(rows, 512))
            fidx += 1
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            total_frames += n
            total_s += dt
            per_step.append(dt)
        if total_s > args.ref_budget_s:
            break
    fps = total_frames / total_s
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": len(per_step), "warmup": args.warmup, "ms_per_step": 1e3 * total_s / max(len(per_step), 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config}: 1 stream, B={B}, 1088x608 heads, "
                                                    f"{gen.cfg.objects[0]} objects"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port",
                         "sample": f"{total_frames} consecutive frames of the {args.config} stream "
                                   f"(oracle decode + restated Tracker.step, OPENBLAS_NUM_THREADS=1)"},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2011_03910_b200 as p
    from paper_2011_03910_b200 import _lib, synth

    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist

    def barrier():
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    B, K, W = args.batch, args.steps, args.warmup
    gen = synth.make(args.config, device=dev, seed=args.seed + rank)
    S = gen.cfg.streams
    batches = [gen.next_batch(B) for _ in range(W + K)]
    torch.cuda.synchronize()
    F = S * B
    cap = p.Capacity(streams=S, max_frames=F, max_candidates=512, max_detections=256, max_tracks=256)
    bt = p.BatchTracker(S, frames_per_update=B, capacity=cap)
    eng = bt.engine
    lib = eng.lib
    stream = torch.cuda.current_stream()

    for i in range(W):
        bt.update(batches[i], trace=False, sync=False)
    eng.finish()
    # counts for algorithmic bytes: one traced pass over the timed batches on a twin tracker
    twin = p.BatchTracker(S, frames_per_update=B, capacity=cap)
    cand, kept, recs = 0, 0, 0
    for i in range(W + K):
        r = twin.update(batches[i], trace=True)
        if i >= W:
            tr = twin.trace(F)
            cand += int(tr["cand_count"].sum())
            kept += int(tr["det_count"].sum())
            recs += int(r.count.sum())
    del twin

    lib.tf_set_profiling(eng.ctx, 1)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    with ClockSampler(local) as clocks:
        start.record(stream)
        for i in range(W, W + K):
            bt.update(batches[i], trace=False, sync=False)
        end.record(stream)
        end.synchronize()
    eng.finish()
    barrier()
    ms = start.elapsed_time(end)
    import ctypes as C
    fr_ms, as_ms, nup = C.c_double(), C.c_double(), C.c_int64()
    lib.tf_kernel_times(eng.ctx, C.byref(fr_ms), C.byref(as_ms), C.byref(nup))
    import numpy as _np
    phase = _np.zeros(32, _np.int64)
    lib.tf_phase_stats(eng.ctx, phase.ctypes.data)
    lib.tf_set_profiling(eng.ctx, 0)

    # ---- end to end through the C ABI with pinned host buffers --------------
    e2e_steps = min(K, args.e2e_steps)
    host_batches = []
    for i in range(1 + e2e_steps):
        src = batches[i]
        host_batches.append(p.HeadOutputs(
            tuple(h.cpu().pin_memory() for h in src.heads),
            tuple(e.cpu().contiguous(memory_format=torch.channels_last).pin_memory() for e in src.embs)))
    bt2 = p.BatchTracker(S, frames_per_update=B, capacity=cap)
    hout = bt2.host_output(F)
    bt2.update(host_batches[0], host_out=hout)            # warm-up (allocates staging)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    for i in range(1, 1 + e2e_steps):
        bt2.update(host_batches[i], host_out=hout, sync=False)
    e1.record(stream)
    e1.synchronize()
    bt2.engine.finish()
    barrier()
    e2e_ms = e0.elapsed_time(e1)
    D = 512
    h2d = F * CONF_BYTES + (cand / K) * (16 + 4 * D) + 8 * F
    d2h = 4 * F + F * cap.max_detections * (8 + 32 + 8)

    # ---- max over ranks, metrics gather (the only collective) ----------------
    local_metrics = torch.tensor([ms, e2e_ms, float(K * F), float(e2e_steps * F), fr_ms.value, as_ms.value,
                                  float(cand), float(kept), float(recs)], dtype=torch.float64, device=dev)
    if pg:
        gathered = [torch.zeros_like(local_metrics) for _ in range(world)]
        pg.all_gather(gathered, local_metrics)
        allm = torch.stack(gathered).cpu().numpy()
    else:
        allm = local_metrics.cpu().numpy()[None]
    if rank == 0:
        max_ms, max_e2e = float(allm[:, 0].max()), float(allm[:, 1].max())
        frames_all, e2e_frames_all = float(allm[:, 2].sum()), float(allm[:, 3].sum())
        value = frames_all / (max_ms / 1e3)
        e2e = e2e_frames_all / (max_e2e / 1e3)
        peak, peak_kind = peaks()
        # associate_kernel algorithmic bytes per launch:
        # per frame 4*D*K det embeddings read + 2*4*D*M track embeddings read+written
        # (~M = K at steady state) + 48 B per record + 40 B per detection (meas, obj).
        kpf = kept / (K * F)
        rpf = recs / (K * F)
        assoc_bytes_launch = F * (4 * D * kpf + 2 * 4 * D * kpf + 48 * rpf + 40 * kpf)
        assoc_launch_ms = as_ms.value / max(nup.value, 1)
        frame_bytes_launch = F * (CONF_BYTES + (cand / (K * F)) * (16 + 4 * D) + 4 * D * kpf + 40 * kpf)
        frame_launch_ms = fr_ms.value / max(nup.value, 1)
        achieved = assoc_bytes_launch / (assoc_launch_ms / 1e3) / 1e9
        traffic = None
        tf = ROOT / "profiles" / "traffic.json"
        if tf.exists():
            traffic = json.loads(tf.read_text()).get(args.config, {}).get("associate_kernel")
        cpu = None
        if not args.no_cpu:
            fps_cpu, n_cpu = cpu_reference_fps(host_frame_iter(batches, args.cpu_frames), args.ref_budget_s)
            cpu = {"value": fps_cpu, "unit": "frames/s", "cores": 1, "kind": "port",
                   "sample": f"first {n_cpu} frames of this rank-0 {args.config} stream (oracle decode + restated "
                             f"Tracker.step, OPENBLAS_NUM_THREADS=1, one core: frames of a stream are sequential)"}
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: 1 stream per GPU, B={B} frames per update, 1088x608 "
                                   f"3-scale JDE heads + 512-d embedding maps, {gen.cfg.objects[0]} objects",
                       "frames_per_step": F * world, "inputs_exceed_l2": True,
                       "l2_policy": "each step reads a fresh 930 MB batch (> 126 MB L2); no flush needed",
                       "parallelism": f"streams sharded, {world} rank(s)"},
            "e2e": {"value": e2e, "unit": "frames/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "steps": e2e_steps},
            "roofline": {"bound": "hbm", "kernel": "associate_kernel", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_launch": assoc_bytes_launch, "ms_per_launch": assoc_launch_ms,
                         "note": "latency-bound sequential association (one CTA per stream); see DESIGN.md"},
            "kernels": {
                "frame_heads_kernel": {"ms_per_launch": frame_launch_ms, "bytes_per_launch": frame_bytes_launch,
                                       "GBps": frame_bytes_launch / (frame_launch_ms / 1e3) / 1e9,
                                       "frac": frame_bytes_launch / (frame_launch_ms / 1e3) / 1e9 / peak},
                "associate_kernel": {"ms_per_launch": assoc_launch_ms, "share_of_step":
                                     as_ms.value / max(ms, 1e-9)}},
            "per_frame": {"candidates": cand / (K * F), "detections": kpf, "records": rpf},
            "assoc_phases_us_per_frame": {
                name: float(phase[i]) / max(phase[11], 1) / (clocks.summary()["sm_mhz"] or 1965)
                for i, name in list(enumerate(["load_predict", "gate", "csr", "cost", "lap", "match", "update_ema",
                                               "records_births"]))
                + [(16, "lap.components_tiecheck"), (17, "lap.peeling"), (18, "lap.residual_setup"),
                   (19, "lap.warp_solves"), (20, "lap.full_restatement")]},
            "assoc_counters_per_frame": {name: float(phase[i]) / max(phase[11], 1) for i, name in
                                         [(8, "tie_fallback"), (9, "finite_entries"), (10, "multi_components"),
                                          (14, "residual_entries"),
                                          (12, "tracks"), (13, "detections")]},
            "gpu_launches": 2 * K,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if pg:
        pg.barrier()
        pg.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg1")
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--cpu-frames", type=int, default=640)
    ap.add_argument("--ref-budget-s", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
