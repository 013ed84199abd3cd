"""Benchmark: tracked frames/sec (decode + NMS + association) on B200 vs the CPU reference.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1] [--impl ours|reference]

A *step* is one ``update(head_outputs)`` of the hot path over one batch of
synthetic head tensors of BASELINE shape (1088x608, three scales, 512-d
embedding maps; paper_2011_03910_b200/synth.py):

* config 1 (default; the BASELINE metric's config): one stream, 50 objects,
  B = 32 consecutive frames per step. Under torchrun every rank runs its own
  stream (weak scaling, no data-path collective).
* configs 3 / 4: 64 / 512 streams x B = 8 frames, sharded over the ranks
  (strong scaling: total work fixed).

Only the final per-rank metrics are gathered (NCCL all_gather, dist.py).

* ``value``   device-resident throughput: CUDA events around the K timed steps
              on the launching stream, barrier + synchronize on both sides,
              max over ranks. Each step reads a fresh batch (>= 233 MB, larger
              than the 126 MB L2), so no L2 flush is needed. When all steps do
              not fit in HBM (config 4 on one GPU) batches are generated between
              steps and each step is timed alone (events), summed.
* ``e2e``     the same update through the C ABI with pinned HOST inputs and
              host outputs, copies inside the timed region.
* ``roofline`` dominant kernel (associate_kernel), algorithmic bytes per launch
              / its CUDA-event duration, against MEASURED_PEAKS.json.
* ``cpu_baseline`` the CPU oracle port of the reference path (decode oracle +
              Tracker.step restatement, OPENBLAS_NUM_THREADS=1), rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes as C
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
CONF_BYTES = 8 * 4 * N_CELLS                    # 434,112 B/frame: the 8 conf planes per scale set
FRAME_BYTES = 24 * 4 * N_CELLS + 512 * 4 * N_CELLS   # 29.1 MB resident per frame
D = 512

# per-config device capacities (smem of the association CTA scales with them)
CAPS = {
    "cfg0": dict(max_candidates=512, max_detections=256, max_tracks=256),
    "cfg1": dict(max_candidates=512, max_detections=256, max_tracks=256),
    "cfg2": dict(max_candidates=768, max_detections=224, max_tracks=384),
    "cfg3": dict(max_candidates=256, max_detections=160, max_tracks=256),
    "cfg4": dict(max_candidates=192, max_detections=96, max_tracks=160),
}


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    LABELS = {"nvmlClocksThrottleReasonHwSlowdown": "hw_slowdown",
              "nvmlClocksThrottleReasonHwThermalSlowdown": "hw_thermal_slowdown",
              "nvmlClocksThrottleReasonSwThermalSlowdown": "sw_thermal_slowdown",
              "nvmlClocksThrottleReasonSwPowerCap": "sw_power_cap"}

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
        bits = {getattr(N, k, None): v for k, v in self.LABELS.items()}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, label in bits.items():
                    if bit and r & bit:
                        self.reasons.add(label)
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


# ---------------------------------------------------------------------------- CPU reference port
def _oracle_stream(frames, limit_s=None):
    """Decode oracle + oracle Tracker.step over one stream's host frames."""
    from oracle import heads as oh
    from oracle import tracker as ot

    trk = ot.OracleTracker(ot.Settings())
    n, t0 = 0, time.perf_counter()
    for i, (heads, embs) in enumerate(frames):
        _, rows = oh.decode_frame(heads, embs)
        trk.step(i, ot.rows_to_dets(rows, D))
        n += 1
        if limit_s and time.perf_counter() - t0 > limit_s:
            break
    return n, time.perf_counter() - t0


def _cpu_worker(args):
    """One process = one stream of the config, generated on the CPU."""
    name, seed, frames, warm = args
    import torch

    torch.set_num_threads(1)
    from paper_2011_03910_b200 import synth

    gen = synth.make(name, device="cpu", seed=seed, streams=1)
    out = gen.next_batch(warm + frames)
    host = [([h[b].numpy() for h in out.heads], [e[b].numpy() for e in out.embs]) for b in range(warm + frames)]
    _oracle_stream(host[:warm])
    n, s = _oracle_stream(host[warm:])
    return n, s


def cpu_baseline_multistream(name: str, seed: int, per_stream_frames: int, workers: int):
    """Process pool, one stream per worker: aggregate frames/s."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        t0 = time.perf_counter()
        res = pool.map(_cpu_worker, [(name, seed + 1000 + i, per_stream_frames, 3) for i in range(workers)])
        wall = time.perf_counter() - t0
    frames = sum(n for n, _ in res)
    busy = max(s for _, s in res)
    return frames / busy, frames, wall


def host_frame_iter(batches, limit):
    n = 0
    for out in batches:
        for b in range(out.frames):
            if n >= limit:
                return
            yield [h[b].cpu().numpy() for h in out.heads], [e[b].cpu().numpy() for e in out.embs]
            n += 1


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    from paper_2011_03910_b200.dist import env

    world, rank, _ = env()
    if rank != 0:
        return
    from paper_2011_03910_b200 import synth

    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.batch
    if cfg.streams == 1:
        gen = synth.make(args.config, device="cpu", seed=args.seed)
        from oracle import heads as oh
        from oracle import tracker as ot

        trk = ot.OracleTracker(ot.Settings())
        fidx, total_frames, total_s, steps = 0, 0, 0.0, 0
        for step in range(args.warmup + args.steps):
            out = gen.next_batch(B)
            frames = [([h[b].numpy() for h in out.heads], [e[b].numpy() for e in out.embs]) for b in range(B)]
            n = B if step >= args.warmup else min(B, 4)
            t0 = time.perf_counter()
            for heads, embs in frames[:n]:
                _, rows = oh.decode_frame(heads, embs)
                trk.step(fidx, ot.rows_to_dets(rows, D))
                fidx += 1
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                total_frames += n
                total_s += dt
                steps += 1
            if total_s > args.ref_budget_s:
                break
        fps, cores = total_frames / total_s, 1
        sample = (f"{total_frames} consecutive frames of the {args.config} stream (oracle decode + restated "
                  f"Tracker.step, OPENBLAS_NUM_THREADS=1; one core: frames of a stream are sequential)")
        ms_step = 1e3 * total_s / max(steps, 1)
    else:
        workers = min(len(os.sched_getaffinity(0)), cfg.streams)
        fps, frames, wall = cpu_baseline_multistream(args.config, args.seed, args.cpu_stream_frames, workers)
        cores, steps = workers, args.steps
        sample = (f"{workers} streams of {args.config} in a {workers}-process pool, {args.cpu_stream_frames} "
                  f"frames each (oracle decode + restated Tracker.step, OPENBLAS_NUM_THREADS=1)")
        ms_step = 1e3 * cfg.streams * B / fps
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if cfg.streams == 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg.streams} stream(s), B={B}, 1088x608 heads, "
                               f"objects {cfg.objects}"},
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- our arm
def tracking_quality(args, cfg_name, S, B, cap, dev, steps=8):
    """MOTA / IDF1 of the GPU outputs of stream 0 against the generator's
    ground truth, scored by the GPU moteval; a fresh,
    untimed run of `steps` updates with its own seed."""
    import paper_2011_03910_b200 as p
    from paper_2011_03910_b200 import moteval, synth
    from paper_2011_03910_b200.tracker import TrackerOutput

    gen = synth.make(cfg_name, device=dev, seed=args.seed + 1000, streams=S)
    gen.record_truth()
    bt = p.BatchTracker(S, tracker_config(args), frames_per_update=B, capacity=cap)
    outs = []
    for i in range(steps):
        batch = gen.next_batch(B)
        if args.dtype == "f16":
            batch = batch.half()
        r = bt.update(batch)
        outs += [TrackerOutput(frame_index=int(r.frame_index[b]), records=r.records(0, b)) for b in range(B)]
        del batch
    rep = moteval.evaluate(gen.truth_frames(0), moteval.outputs_to_frames(outs))
    return {"stream": 0, "frames": len(outs), "iou_min": 0.5, "MOTA": rep.mota, "IDF1": rep.idf1,
            "MOTP": rep.motp, "IDs": rep.id_switches, "FP": rep.fp, "FN": rep.fn, "scorer": "GPU moteval"}


def tracker_config(args):
    """TrackerConfig of the run: the reference path, or the JDE extensions (--jde)."""
    import paper_2011_03910_b200 as p
    if getattr(args, "jde", False):
        return p.TrackerConfig(motion_lambda=0.98, iou_stage=True, iou_threshold=0.5)
    return p.TrackerConfig()


def run_ours(args):
    import numpy as np
    import torch

    from paper_2011_03910_b200.dist import env, gather_metrics, shard_streams, summarize

    world, rank, local = env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    import paper_2011_03910_b200 as p
    from paper_2011_03910_b200 import synth

    dist = None
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=dev)
        dist = tdist

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.batch
    multi = cfg.streams > 1
    S = shard_streams(cfg.streams, world, rank).n_streams if multi else 1
    K, W = args.steps, args.warmup
    F = S * B
    gen = synth.make(args.config, device=dev, seed=args.seed + rank, streams=S)
    cap = p.Capacity(streams=S, max_frames=F, **CAPS[args.config])
    free, _ = torch.cuda.mem_get_info(dev)
    esz = 2 if args.dtype == "f16" else 4          # input element bytes (f16: MIXED input mode)
    conf_bytes = CONF_BYTES * esz // 4
    step_bytes = F * FRAME_BYTES * esz // 4

    def gen_batch():
        b = gen.next_batch(B)
        return b.half() if args.dtype == "f16" else b
    streamed = (W + K) * step_bytes > 0.55 * free
    batches = None if streamed else [gen_batch() for _ in range(W + K)]
    torch.cuda.synchronize()

    pipe = not (streamed or args.no_pipeline)
    bt = p.BatchTracker(S, tracker_config(args), frames_per_update=B, capacity=cap, pipeline=pipe)
    eng, lib = bt.engine, bt.engine.lib
    stream = torch.cuda.current_stream()

    def batch(i):
        return gen_batch() if streamed else batches[i]

    for i in range(W):
        bt.update(batch(i), trace=streamed, sync=False)
    eng.finish()

    cand = kept = recs = 0
    if not streamed:
        # counts for the algorithmic bytes: one traced pass on a twin tracker
        twin = p.BatchTracker(S, tracker_config(args), frames_per_update=B, capacity=cap)
        for i in range(W + K):
            r = twin.update(batches[i], trace=True)
            if i >= W:
                tr = twin.trace(F)
                cand += int(tr["cand_count"].sum())
                kept += int(tr["det_count"].sum())
                recs += int(r.count.sum())
        del twin

    # kernel events in the timed region; the in-kernel phase timers (level 2)
    # only in the separate diagnostic pass below (streamed runs keep them on)
    # events on every prof_stride-th update: their host cost would otherwise
    # show in small-batch runs (B = 1: ~6 event records per 30 us update)
    prof_stride = max(1, 8 // B)
    lib.tf_set_profiling(eng.ctx, (2 if streamed else 1) | (prof_stride << 4))
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = 0.0
    barrier()
    with ClockSampler(local) as clocks:
        if not streamed:
            e_start.record(stream)
            for i in range(W, W + K):
                bt.update(batches[i], trace=False, sync=False)
            bt.join()                      # the timed region ends after the last association
            e_end.record(stream)
            e_end.synchronize()
            ms = e_start.elapsed_time(e_end)
        else:
            for i in range(W, W + K):
                nb = batch(i)
                torch.cuda.synchronize()
                e_start.record(stream)
                r = bt.update(nb, trace=True, sync=False)
                e_end.record(stream)
                e_end.synchronize()
                ms += e_start.elapsed_time(e_end)
                tr = bt.trace(F)
                cand += int(tr["cand_count"].sum())
                kept += int(tr["det_count"].sum())
                recs += int(r.count.sum())
                del nb
    eng.finish()
    barrier()
    fr_ms, as_ms, nup = C.c_double(), C.c_double(), C.c_int64()
    lib.tf_kernel_times(eng.ctx, C.byref(fr_ms), C.byref(as_ms), C.byref(nup))
    phase = np.zeros(32, np.int64)
    lib.tf_phase_stats(eng.ctx, phase.ctypes.data)
    lib.tf_set_profiling(eng.ctx, 0)
    if not streamed:
        # per-phase breakdown of the association: the same batches on a fresh
        # tracker with the phase timers on, outside the timed region
        pbt = p.BatchTracker(S, tracker_config(args), frames_per_update=B, capacity=cap, pipeline=pipe)
        lib.tf_set_profiling(pbt.engine.ctx, 2)
        for i in range(W + K):
            pbt.update(batches[i], trace=False, sync=False)
        pbt.join()
        pbt.engine.finish()
        lib.tf_phase_stats(pbt.engine.ctx, phase.ctypes.data)
        lib.tf_set_profiling(pbt.engine.ctx, 0)
        del pbt

    # ---- end to end through the C ABI with pinned host buffers --------------
    e2e_steps = min(K, args.e2e_steps)
    e2e_ms, e2e_reason, e2e_kernels = None, None, None
    if (1 + e2e_steps) * step_bytes > args.e2e_host_gb * 2**30 or streamed:
        e2e_reason = f"pinned host copy of {1 + e2e_steps} steps ({(1 + e2e_steps) * step_bytes / 2**30:.0f} GiB) " \
                     f"exceeds the {args.e2e_host_gb} GiB budget"
    else:
        host_batches = [p.HeadOutputs(
            tuple(h.cpu().pin_memory() for h in batches[i].heads),
            tuple(e.cpu().contiguous(memory_format=torch.channels_last).pin_memory() for e in batches[i].embs))
            for i in range(1 + e2e_steps)]
        bt2 = p.BatchTracker(S, tracker_config(args), frames_per_update=B, capacity=cap, pipeline=pipe)
        hout = bt2.host_output(F)
        bt2.update(host_batches[0], host_out=hout)            # warm-up (allocates staging)
        barrier()
        lib.tf_set_profiling(bt2.engine.ctx, 1 | (prof_stride << 4))
        e_start.record(stream)
        for i in range(1, 1 + e2e_steps):
            bt2.update(host_batches[i], host_out=hout, sync=False)
        bt2.join()                         # ... and after the last records reached host memory
        e_end.record(stream)
        e_end.synchronize()
        bt2.engine.finish()
        barrier()
        e2e_ms = e_start.elapsed_time(e_end)
        tl = np.zeros(6 * 64)
        ntl = C.c_int32()
        lib.tf_timeline(bt2.engine.ctx, tl.ctypes.data, 64, C.byref(ntl))
        tl = tl[:6 * min(ntl.value, 64)].reshape(-1, 6)
        f2, a2, n2 = C.c_double(), C.c_double(), C.c_int64()
        lib.tf_kernel_times(bt2.engine.ctx, C.byref(f2), C.byref(a2), C.byref(n2))
        h2 = C.c_double()
        lib.tf_copy_times(bt2.engine.ctx, C.byref(h2))
        e2e_kernels = {"h2d_ms_per_step": h2.value / max(n2.value, 1),
                       "frame_heads_ms_per_launch": f2.value / max(n2.value, 1),
                       "associate_ms_per_launch": a2.value / max(n2.value, 1), "launches": n2.value,
                       "assoc_gap_ms_mean": float(np.mean(tl[1:, 2] - tl[:-1, 3])) if len(tl) > 1 else None,
                       "timeline_ms": [[round(float(v), 3) for v in row] for row in tl[:4]]}
        lib.tf_set_profiling(bt2.engine.ctx, 0)
        del host_batches
    h2d = F * conf_bytes + (cand / K) * esz * (4 + D) + 8 * F
    d2h = 4 * F + F * cap.max_detections * (8 + 32 + 8)

    # ---- max over ranks: the run's only collective ---------------------------
    ex = bt.export(0)
    per_rank = gather_metrics({"frames": float(K * F), "ids_issued": float(ex["next_id"] - 1),
                               "live_tracks": float(ex["count"]), "candidates": float(cand),
                               "detections": float(kept), "records": float(recs), "elapsed_ms": ms}, device=dev)
    e2e_all = gather_metrics({"frames": float(e2e_steps * F), "elapsed_ms": e2e_ms or 0.0}, device=dev)
    if rank == 0:
        summ = summarize(per_rank)
        value = summ["frames_per_s"]
        e2e_value = summarize(e2e_all)["frames_per_s"] if e2e_ms else None
        max_ms = summ["max_elapsed_ms"]
        peak, peak_kind = peaks()
        kpf, rpf, cpf = kept / (K * F), recs / (K * F), cand / (K * F)
        # associate_kernel algorithmic bytes per launch: per
        # frame 4*D*K detection embeddings + 2*4*D*K track embeddings (EMA read +
        # write) + 48 B per record + 40 B per detection
        assoc_bytes_launch = F * (4 * D * kpf + 2 * 4 * D * kpf + 48 * rpf + 40 * kpf)
        assoc_launch_ms = as_ms.value / max(nup.value, 1)
        frame_bytes_launch = F * (conf_bytes + cpf * esz * (4 + D) + 4 * D * kpf + 40 * kpf)
        frame_launch_ms = fr_ms.value / max(nup.value, 1)
        a_gbs = assoc_bytes_launch / (assoc_launch_ms / 1e3) / 1e9
        f_gbs = frame_bytes_launch / (frame_launch_ms / 1e3) / 1e9
        dominant = "associate_kernel" if as_ms.value >= fr_ms.value else "frame_heads_kernel"
        traffic = None
        tfile = ROOT / "profiles" / "traffic.json"
        if tfile.exists():
            traffic = json.loads(tfile.read_text()).get(args.config, {}).get(dominant)
        quality = None
        if not streamed:
            quality = tracking_quality(args, args.config, S, B, cap, dev)
        cpu = None
        if not args.no_cpu:
            if not multi:
                n_cpu, s_cpu = _oracle_stream(host_frame_iter(batches or [], args.cpu_frames), args.ref_budget_s)
                cpu = {"value": n_cpu / s_cpu, "unit": "frames/s", "cores": 1, "kind": "port",
                       "sample": f"first {n_cpu} frames of this rank-0 {args.config} stream (oracle decode + "
                                 f"restated Tracker.step, OPENBLAS_NUM_THREADS=1, one core: frames of a stream "
                                 f"are sequential)"}
            else:
                workers = min(len(os.sched_getaffinity(0)), cfg.streams)
                fps_cpu, n_cpu, _ = cpu_baseline_multistream(args.config, args.seed, args.cpu_stream_frames, workers)
                cpu = {"value": fps_cpu, "unit": "frames/s", "cores": workers, "kind": "port",
                       "sample": f"{workers} streams x {args.cpu_stream_frames} frames of {args.config}, one "
                                 f"stream per process (synthetic, generated on the CPU with the same config)"}
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "strong" if multi else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg.streams if multi else 1} stream(s) "
                                   f"{'sharded over' if multi else 'per'} GPU(s), B={B} frames per stream per "
                                   f"update, 1088x608 3-scale JDE heads + 512-d embedding maps, objects "
                                   f"{cfg.objects}",
                       "frames_per_step": F * world if not multi else cfg.streams * B,
                       "input_dtype": "fp16 (MIXED input mode)" if args.dtype == "f16" else "fp32",
                       "streams_per_rank": S, "inputs_exceed_l2": True,
                       "l2_policy": f"each step reads a fresh {step_bytes / 2**20:.0f} MB batch (> 126 MB L2)",
                       "generation": "streamed between steps, steps timed one by one" if streamed
                       else "pre-generated on device",
                       "pipeline": "decode of step i+1 overlaps association of step i" if pipe else "off",
                       "parallelism": f"streams sharded over {world} rank(s), final NCCL all_gather",
                       "tracker": "jde-extensions (lambda 0.98, IoU stage 0.5)" if args.jde else "reference"},
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps if e2e_ms else 0,
                    "kernels": e2e_kernels,
                    **({"unavailable": e2e_reason} if e2e_reason else {})},
            "roofline": {"bound": "hbm", "kernel": dominant,
                         "achieved": a_gbs if dominant == "associate_kernel" else f_gbs, "peak": peak,
                         "unit": "GB/s",
                         "frac": (a_gbs if dominant == "associate_kernel" else f_gbs) / peak,
                         "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_launch": assoc_bytes_launch if dominant == "associate_kernel"
                         else frame_bytes_launch,
                         "ms_per_launch": assoc_launch_ms if dominant == "associate_kernel" else frame_launch_ms,
                         "note": "association is a per-stream dependency chain (latency-bound); DESIGN.md s6"},
            "kernels": {
                "event_sample_stride": prof_stride,   # CUDA events on every N-th timed update
                "frame_heads_kernel": {"ms_per_launch": frame_launch_ms, "bytes_per_launch": frame_bytes_launch,
                                       "GBps": f_gbs, "frac": f_gbs / peak},
                "associate_kernel": {"ms_per_launch": assoc_launch_ms, "bytes_per_launch": assoc_bytes_launch,
                                     "GBps": a_gbs, "frac": a_gbs / peak,
                                     "share_of_step": as_ms.value / max(ms, 1e-9)}},
            "per_frame": {"candidates": cpf, "detections": kpf, "records": rpf},
            "assoc_phases_us_per_frame": {
                name: float(phase[i]) / max(phase[11], 1) / (clocks.summary()["sm_mhz"] or 1965)
                for i, name in list(enumerate(["load_predict", "gate", "csr", "cost", "lap", "match",
                                               "update_ema", "records_births"]))
                + [(16, "lap.components_tiecheck"), (17, "lap.peeling"), (18, "lap.residual_setup"),
                   (19, "lap.warp_solves"), (20, "lap.full_restatement"), (21, "cost.s1_wait"),
                   (22, "cost.leader_work"), (23, "cost.s2_wait"), (24, "cost.ema_wait"), (25, "cost.go_signal"),
                   (26, "ema_signal"), (30, "births_tail"), (31, "whole_frame"),
                   (28, "launch.prologue"), (29, "launch.epilogue")]},
            "assoc_counters_per_frame": {name: float(phase[i]) / max(phase[11], 1) for i, name in
                                         [(8, "tie_fallback"), (9, "finite_entries"), (10, "multi_components"),
                                          (14, "residual_entries"), (12, "tracks"), (13, "detections"), (15, "peel_rounds")]},
            "ranks": per_rank,
            "gpu_launches": 2 * K * (1 if not streamed else 1) + (K if streamed else 0),
            "clocks": clocks.summary(),
            "quality": quality,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg1", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--batch", type=int, default=None, help="frames per stream per update (default: config's B)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-host-gb", type=float, default=24.0)
    ap.add_argument("--cpu-frames", type=int, default=640)
    ap.add_argument("--cpu-stream-frames", type=int, default=40)
    ap.add_argument("--ref-budget-s", type=float, default=20.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true", help="serialise decode and association")
    ap.add_argument("--jde", action="store_true",
                    help="JDE extensions on (lambda = 0.98 fused cost, IoU second stage at 0.5); off = reference path")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f16"],
                    help="head / embedding input type (f16 = MIXED-precision input mode, SURVEY 8(f))")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
