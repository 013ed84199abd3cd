"""Benchmark: tracked frames/sec (decode + NMS + association) on B200 vs the CPU reference.

Contract (one JSON line on rank 0):
  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg1] [--impl ours|reference]

``--gpus N`` with N > 1 outside torchrun re-launches itself under
``torch.distributed.run`` with N ranks (one GPU each, NCCL); under torchrun
WORLD_SIZE must equal N.

A *step* is one ``update(head_outputs)`` of the hot path over one batch of
synthetic head tensors of BASELINE shape (1088x608, three scales, 512-d
embedding maps; paper_2011_03910_b200/synth.py):

* config 1 (default; the BASELINE metric's config): one stream per GPU, 50
  objects, B = 32 consecutive frames per step (weak scaling: each rank tracks
  its own stream, no data-path collective).
* configs 3 / 4: 64 / 512 streams x B = 8 frames, sharded over the ranks
  (strong scaling: total work fixed). The default cfg1 run also carries a
  ``cfg4`` block measured the same way at every N (512 streams sharded).

Only the final per-rank metrics are gathered (NCCL all_gather, dist.py).

* ``value``    device-resident throughput: CUDA events around the K timed steps
               on the launching stream, barrier + synchronize on both sides,
               max over ranks. Each step reads a fresh batch (>= 233 MB, larger
               than the 126 MB L2), so no L2 flush is needed. When all steps do
               not fit in HBM (config 4 on one GPU) batches are generated between
               steps and each step is timed alone (events), summed.
* ``e2e``      the same update through the C ABI with pinned HOST inputs and
               host outputs, copies inside the timed region.
* ``roofline`` dominant kernel (associate_kernel): SURVEY 8(d) algorithmic bytes
               per frame x frames per launch / its CUDA-event duration, against
               MEASURED_PEAKS.json; ``step`` = the same bytes over the whole step.
* ``parity``   rank 0: the CPU oracle (decode oracle + restated Tracker.step) on
               every frame the GPU processed (warm-up and timed steps), compared
               with the GPU records and association trace frame by frame.
* ``cpu_baseline`` that oracle run's throughput (N = 1, rank 0, one core).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import socket
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
FRAME_BYTES = 24 * 4 * N_CELLS + 512 * 4 * N_CELLS   # 29.1 MB resident per frame (fp32)
D = 512
REF_DIR = ROOT / "baseline" / "_ref"

# per-config device capacities (smem of the association CTA scales with them)
CAPS = {
    "cfg0": dict(max_candidates=512, max_detections=256, max_tracks=256),
    "cfg1": dict(max_candidates=512, max_detections=256, max_tracks=256),
    "cfg2": dict(max_candidates=768, max_detections=224, max_tracks=384),
    "cfg3": dict(max_candidates=256, max_detections=160, max_tracks=256),
    "cfg4": dict(max_candidates=192, max_detections=96, max_tracks=160),
}


def alg_bytes(frames: float, esz: int, cand: float, kept: float, recs: float) -> float:
    """SURVEY 8(d) algorithmic bytes of `frames` frames with `cand` candidates,
    `kept` detections and `recs` records in total: the compulsory conf planes
    (8 per scale set), the candidates' deltas, the gathered embeddings and the
    written records; input terms scale with the input element size `esz`
    (2 for the MIXED fp16 input mode)."""
    return frames * 8 * esz * N_CELLS + 16 * esz / 4 * cand + esz * D * kept + 48 * recs


def peaks():
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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


def workload_config(args, world: int) -> dict:
    """The workload both arms measure (identical dict in both JSON lines)."""
    from paper_2011_03910_b200 import synth

    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.batch
    multi = cfg.streams > 1
    esz = 2 if args.dtype == "f16" else 4
    return {
        "workload": f"{args.config}: {cfg.streams if multi else 1} stream(s) {'sharded over' if multi else 'per'} "
                    f"GPU(s), B={B} frames per stream per update, 1088x608 3-scale JDE heads + 512-d embedding "
                    f"maps, objects {cfg.objects}",
        "frames_per_step": (cfg.streams if multi else world) * B,
        "input_dtype": "fp16 (MIXED input mode)" if args.dtype == "f16" else "fp32",
        "seed": args.seed,
        "inputs": "seeded synthetic head tensors generated on the GPU (same generator, seed and draws in both arms)",
        "inputs_exceed_l2": True,
        "l2_policy": f"each step reads a fresh {FRAME_BYTES * esz // 4 * B / 2**20:.0f} MB-per-stream batch "
                     f"(> 126 MB L2)",
        "tracker": "jde-extensions (lambda 0.98, IoU stage 0.5)" if args.jde else "reference",
    }


# ---------------------------------------------------------------------------- CPU sides
def _frames_to_host(batch, frames):
    """Numpy copies of the given frames of a HeadOutputs batch (per-scale
    [24,H,W] / [D,H,W])."""
    import torch

    idx = torch.as_tensor(list(frames), dtype=torch.long, device=batch.heads[0].device)
    heads = [h.index_select(0, idx).float().cpu().numpy() for h in batch.heads]
    embs = [e.index_select(0, idx).float().cpu().contiguous().numpy() for e in batch.embs]
    return [([h[i] for h in heads], [e[i] for e in embs]) for i in range(len(idx))]


def _reference_tracker():
    """The unmodified reference (baseline/_ref, pip-installed from
    /root/reference) when present: (parse_output, Tracker) and "reference";
    otherwise the oracle port and "port"."""
    if (REF_DIR / "trackforge" / "tracker.py").exists():
        sys.path.insert(0, str(REF_DIR))
        from trackforge.postproc import parse_output
        from trackforge.tracker import Tracker, TrackerConfig
        return (lambda: Tracker(TrackerConfig())), (lambda rows: parse_output(rows, D)), "reference"
    from oracle import tracker as ot
    return (lambda: ot.OracleTracker(ot.Settings())), (lambda rows: ot.rows_to_dets(rows, D)), "port"


def _cpu_worker(args):
    """One process = one stream of a multi-stream config, generated on the CPU."""
    name, seed, frames, warm = args
    import torch

    torch.set_num_threads(1)
    from oracle import heads as oh
    from paper_2011_03910_b200 import synth

    make, parse, _ = _reference_tracker()
    gen = synth.make(name, device="cpu", seed=seed, streams=1)
    out = gen.next_batch(warm + frames)
    host = [([h[b].numpy() for h in out.heads], [e[b].numpy() for e in out.embs]) for b in range(warm + frames)]
    trk = make()
    for i, (h, e) in enumerate(host[:warm]):
        trk.step(i, parse(oh.decode_frame(h, e)[1]))
    t0 = time.perf_counter()
    for i, (h, e) in enumerate(host[warm:]):
        trk.step(warm + i, parse(oh.decode_frame(h, e)[1]))
    return frames, time.perf_counter() - t0


def cpu_multistream(name: str, seed: int, per_stream_frames: int, workers: int):
    """Process pool, one stream per worker: aggregate frames/s."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    with ctx.Pool(workers) as pool:
        res = pool.map(_cpu_worker, [(name, seed + 1000 + i, per_stream_frames, 8) for i in range(workers)])
    frames = sum(n for n, _ in res)
    busy = max(s for _, s in res)
    return frames / busy, frames


# ---------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's CPU implementation of the path on the box's host cores,
    on the same workload, inputs and config dict as our arm. Rank 0 only."""
    from paper_2011_03910_b200.dist import env

    world, rank, _ = env()
    if rank != 0:
        return
    import torch

    from oracle import heads as oh
    from paper_2011_03910_b200 import synth

    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.batch
    make, parse, kind = _reference_tracker()
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    if cfg.streams == 1:
        # exactly our arm's rank-0 inputs: same generator, seed and device
        gen = synth.make(args.config, device=dev, seed=args.seed)
        trk = make()
        fidx, total_frames, total_s, steps = 0, 0, 0.0, 0
        for step in range(args.warmup + args.steps):
            batch = gen.next_batch(B)
            if args.dtype == "f16":
                batch = batch.half()
            frames = _frames_to_host(batch, range(B))
            del batch
            t0 = time.perf_counter()
            for heads, embs in frames:          # every frame of every step, warm-up included (contiguous)
                trk.step(fidx, parse(oh.decode_frame(heads, embs)[1]))
                fidx += 1
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                total_frames += B
                total_s += dt
                steps += 1
                if total_s > args.ref_budget_s:
                    break
        fps, cores = total_frames / total_s, 1
        sample = (f"{total_frames} consecutive frames ({steps} steps after {args.warmup} warm-up steps) of the "
                  f"{args.config} stream, our arm's rank-0 inputs (decode oracle + "
                  f"{'the unmodified reference parse_output + Tracker.step' if kind == 'reference' else 'the oracle port of Tracker.step'}"
                  f", OPENBLAS_NUM_THREADS=1; one core: frames of a stream are sequential)")
        ms_step = 1e3 * total_s / max(steps, 1)
    else:
        workers = min(len(os.sched_getaffinity(0)), cfg.streams)
        fps, frames = cpu_multistream(args.config, args.seed, args.cpu_stream_frames, workers)
        cores, steps = workers, args.steps
        sample = (f"{workers} streams of {args.config} in a {workers}-process pool, {args.cpu_stream_frames} "
                  f"frames each after 8 warm-up frames, generated on the CPU with the same config "
                  f"({'unmodified reference' if kind == 'reference' else 'oracle port'}, OPENBLAS_NUM_THREADS=1)")
        ms_step = 1e3 * cfg.streams * B / fps
    line = {
        "impl": "reference", "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
        "steps": steps, "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if cfg.streams == 1 else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload_config(args, world),
        "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": cores, "kind": kind, "sample": sample},
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


def launches(bt) -> int:
    n = C.c_int64()
    bt.engine.lib.tf_launch_count(bt.engine.ctx, C.byref(n))
    return int(n.value)


def parity_check(args, batches, gpu_frames, B) -> dict:
    """The CPU oracle over every frame the GPU processed (one stream, warm-up
    and timed steps in order), compared with the GPU's per-frame records and
    association trace (oracle/compare.py); also times it (cpu_baseline)."""
    from oracle import heads as oh
    from oracle import tracker as ot
    from oracle.compare import FrameCompare

    trk = ot.OracleTracker(ot.Settings())
    cmp = FrameCompare(strict=False)
    busy, f = 0.0, 0
    for batch in batches:
        host = _frames_to_host(batch, range(B))
        for heads, embs in host:
            t0 = time.perf_counter()
            codes, rows = oh.decode_frame(heads, embs)
            tr = trk.step(f, ot.rows_to_dets(rows, D))
            busy += time.perf_counter() - t0
            g = gpu_frames[f]
            k = int(g["det_count"])
            recs = [(int(g["ids"][i]), tuple(g["box"][i]), float(g["obj"][i])) for i in range(int(g["count"]))]
            cmp.check(f, tr, recs, g["code"][:k], g["track"][:k], g["cost"][:k], g["matched"][:k], codes,
                      gpu_cand_count=g["cand"])
            f += 1
        del host
    return cmp.summary(), f, busy


def timed_updates(bt, batches, stream, lib):
    """K updates of pre-generated batches between two events on `stream`."""
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for b in batches:
        bt.update(b, trace=False, sync=False)
    bt.join()                      # the timed region ends after the last association
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1)


def streamed_updates(bt, gen_batch, K, F, stream, trace_counts, host_us=None):
    """K updates of batches generated between steps, each timed alone (events).

    The stream is held (tf_stream_hold) until update() has queued all of its
    work, so the events time the device work of the update, not the host's
    submission of it (~0.1-0.2 ms of Python + C per update at 64-512 streams,
    which a producer that queues ahead hides); the host time is returned in
    ``host_us``."""
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib = bt.engine.lib
    flag = torch.zeros(1, dtype=torch.int32).pin_memory()
    ms = 0.0
    for _ in range(K):
        nb = gen_batch()
        torch.cuda.synchronize()
        flag.zero_()
        bt.engine.check(lib.tf_stream_hold(flag.data_ptr(), stream.cuda_stream), "hold")
        e0.record(stream)
        try:
            t0 = time.perf_counter()
            r = bt.update(nb, trace=True, sync=False)
            if host_us is not None:
                host_us.append(1e6 * (time.perf_counter() - t0))
            e1.record(stream)
        finally:
            flag.fill_(1)                  # release the stream (always)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        tr = bt.trace(F)
        trace_counts[0] += int(tr["cand_count"].sum())
        trace_counts[1] += int(tr["det_count"].sum())
        trace_counts[2] += int(r.count.sum())
        del nb
    return ms


def cfg4_block(args, world, rank, dev, barrier, shard_world=None):
    """Config 4 strong scaling at this N: 512 streams sharded over the ranks,
    B = 8, batches generated between steps and each step timed alone.
    ``shard_world`` > world runs rank 0's shard of a larger job on this GPU
    (the per-GPU work at that many GPUs, e.g. 64 streams for 8)."""
    import torch

    import paper_2011_03910_b200 as p
    from paper_2011_03910_b200 import synth
    from paper_2011_03910_b200.dist import gather_metrics, shard_streams, summarize

    cfg = synth.CONFIGS["cfg4"]
    sh = shard_streams(cfg.streams, shard_world or world, rank)
    S, B = sh.n_streams, cfg.batch
    F = S * B
    gen = synth.make("cfg4", device=dev, seed=args.seed + 7 + rank, streams=S)
    cap = p.Capacity(streams=S, max_frames=F, **CAPS["cfg4"])
    bt = p.BatchTracker(S, tracker_config(args), frames_per_update=F // S, capacity=cap)
    stream = torch.cuda.current_stream()
    counts = [0, 0, 0]
    for _ in range(args.cfg4_warmup):
        nb = gen.next_batch(B)
        bt.update(nb, sync=True)
        del nb
    barrier()
    bt.engine.lib.tf_set_profiling(bt.engine.ctx, 1)
    host_us = []
    ms = streamed_updates(bt, lambda: gen.next_batch(B), args.cfg4_steps, F, stream, counts, host_us)
    f_ms, a_ms, n = C.c_double(), C.c_double(), C.c_int64()
    bt.engine.lib.tf_kernel_times(bt.engine.ctx, C.byref(f_ms), C.byref(a_ms), C.byref(n))
    bt.engine.finish()
    barrier()
    per_rank = gather_metrics({"frames": float(args.cfg4_steps * F), "elapsed_ms": ms,
                               "candidates": float(counts[0]), "detections": float(counts[1]),
                               "records": float(counts[2])}, device=dev)
    summ = summarize(per_rank)
    frames = summ["frames"]
    cand = sum(m["candidates"] for m in per_rank)
    kept = sum(m["detections"] for m in per_rank)
    recs = sum(m["records"] for m in per_rank)
    peak, _ = peaks()
    step_ms = summ["max_elapsed_ms"] / args.cfg4_steps
    # whole-job bytes over the slowest rank's time, against N x HBM peak
    byt = alg_bytes(frames, 4, cand, kept, recs)
    ach = byt / (summ["max_elapsed_ms"] / 1e3) / 1e9
    return {"streams": cfg.streams, "streams_per_rank": S, "B": B, "steps": args.cfg4_steps,
            "warmup": args.cfg4_warmup, "frames_per_s": summ["frames_per_s"], "ms_per_step": step_ms,
            "gpus_active": len(per_rank), "scaling": "strong",
            "timing": "device time of each update with its launches pre-queued (stream held until update() returns)",
            "host_submit_us_per_update": statistics.mean(host_us) if host_us else None,
            "rank0_kernels_ms_per_step": {"frame_heads_kernel": f_ms.value / max(n.value, 1),
                                          "associate_kernel": a_ms.value / max(n.value, 1)},
            "roofline": {"achieved_GBps": ach, "peak_GBps": peak * len(per_rank),
                         "frac": ach / (peak * len(per_rank)),
                         "bytes_per_frame": byt / max(frames, 1)},
            "per_frame": {"candidates": cand / max(frames, 1), "detections": kept / max(frames, 1),
                          "records": recs / max(frames, 1)}}


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
    # rank r's stream: seed + r (rank 0 = the reference arm's inputs)
    gen = synth.make(args.config, device=dev, seed=args.seed + rank, streams=S)
    cap = p.Capacity(streams=S, max_frames=F, **CAPS[args.config])
    free, _ = torch.cuda.mem_get_info(dev)
    esz = 2 if args.dtype == "f16" else 4          # input element bytes (f16: MIXED input mode)
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

    for i in range(W):
        bt.update(gen_batch() if streamed else batches[i], trace=streamed, sync=False)
    eng.finish()

    cand = kept = recs = 0
    gpu_frames = []
    twin_export = None
    if not streamed:
        # counts for the algorithmic bytes and the per-frame outputs for the
        # parity check: one traced pass of the same batches on a twin tracker
        twin = p.BatchTracker(S, tracker_config(args), frames_per_update=B, capacity=cap)
        for i in range(W + K):
            r = twin.update(batches[i], trace=True)
            tr = {k: v.cpu().numpy() for k, v in twin.trace(F).items()}
            cnt, ids = r.count.cpu().numpy(), r.track_id.cpu().numpy()
            box, obj = r.box.cpu().numpy(), r.objectness.cpu().numpy()
            if i >= W:
                cand += int(tr["cand_count"].sum())
                kept += int(tr["det_count"].sum())
                recs += int(cnt.sum())
            for f in range(B):                     # stream 0 of this rank
                gpu_frames.append({"count": cnt[f], "ids": ids[f, :cnt[f]].copy(), "box": box[f, :cnt[f]].copy(),
                                   "obj": obj[f, :cnt[f]].copy(), "cand": tr["cand_count"][f],
                                   "det_count": tr["det_count"][f], "code": tr["det_code"][f].copy(),
                                   "track": tr["det_track"][f].copy(), "cost": tr["det_cost"][f].copy(),
                                   "matched": tr["det_matched"][f].copy()})
        twin_export = twin.export(0)
        del twin

    # kernel events on every prof_stride-th update (their host cost would
    # otherwise show in small-batch runs); phase timers only in the
    # diagnostic pass below
    prof_stride = max(1, 8 // B)
    lib.tf_set_profiling(eng.ctx, (2 if streamed else 1) | (prof_stride << 4))
    barrier()
    n_launch0 = launches(bt)
    with ClockSampler(local) as clocks:
        if not streamed:
            ms = timed_updates(bt, batches[W:W + K], stream, lib)
        else:
            counts = [0, 0, 0]
            ms = streamed_updates(bt, gen_batch, K, F, stream, counts)
            cand, kept, recs = counts
    eng.finish()
    n_launch = launches(bt) - n_launch0
    barrier()
    fr_ms, as_ms, nup = C.c_double(), C.c_double(), C.c_int64()
    lib.tf_kernel_times(eng.ctx, C.byref(fr_ms), C.byref(as_ms), C.byref(nup))
    phase = np.zeros(40, np.int64)
    lib.tf_phase_stats(eng.ctx, phase.ctypes.data)
    lib.tf_set_profiling(eng.ctx, 0)
    same_state = None
    if twin_export is not None:
        ex = bt.export(0)
        same_state = all(np.asarray(ex[k]).tobytes() == np.asarray(twin_export[k]).tobytes() for k in ex)
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
        e2e_ms = timed_updates_host(bt2, host_batches[1:], hout, stream)
        bt2.engine.finish()
        barrier()
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
                       "assoc_gap_ms_mean": float(np.mean(tl[1:, 2] - tl[:-1, 3])) if len(tl) > 1 else None}
        lib.tf_set_profiling(bt2.engine.ctx, 0)
        del host_batches
    h2d = F * 8 * esz * N_CELLS + (cand / K) * esz * (4 + D) + 8 * F
    d2h = 4 * F + F * cap.max_detections * (8 + 32 + 8)

    # ---- the run's only collective: per-rank metrics -------------------------
    ex = bt.export(0)
    per_rank = gather_metrics({"frames": float(K * F), "ids_issued": float(ex["next_id"] - 1),
                               "live_tracks": float(ex["count"]), "candidates": float(cand),
                               "detections": float(kept), "records": float(recs), "elapsed_ms": ms}, device=dev)
    e2e_all = gather_metrics({"frames": float(e2e_steps * F), "elapsed_ms": e2e_ms or 0.0}, device=dev)
    quality = parity = cpu = None
    if rank == 0:
        if not streamed:
            quality = tracking_quality(args, args.config, S, B, cap, dev)
        if not multi and not args.no_cpu and gpu_frames:
            summary, n_cpu, busy = parity_check(args, batches, gpu_frames, B)
            parity = {**summary, "timed_tracker_state_equals_traced": same_state,
                      "scope": f"rank 0's stream, all {n_cpu} frames of the {W} warm-up + {K} timed steps "
                               f"(the timed tracker's final state is compared bit for bit with the traced "
                               f"twin's)"}
            if world == 1:
                cpu = {"value": n_cpu / busy, "unit": "frames/s", "cores": 1, "kind": "port",
                       "sample": f"the {n_cpu} frames of this run's stream (decode oracle + oracle port of "
                                 f"Tracker.step, OPENBLAS_NUM_THREADS=1, one core: frames of a stream are "
                                 f"sequential); the --impl reference arm times the unmodified reference"}
        elif multi and not args.no_cpu and world == 1:
            workers = min(len(os.sched_getaffinity(0)), cfg.streams)
            fps_cpu, _ = cpu_multistream(args.config, args.seed, args.cpu_stream_frames, workers)
            cpu = {"value": fps_cpu, "unit": "frames/s", "cores": workers, "kind": "port",
                   "sample": f"{workers} streams x {args.cpu_stream_frames} frames of {args.config}, one "
                             f"stream per process (synthetic, generated on the CPU with the same config)"}
    c4 = None
    if not args.no_cfg4 and args.config == "cfg1":
        del batches
        torch.cuda.empty_cache()
        c4 = cfg4_block(args, world, rank, dev, barrier)
        if world == 1 and args.cfg4_project:
            # the per-GPU share at 2/4/8 GPUs, measured on this one: rank 0's
            # shard of the 512 streams (no other rank exists; no collective)
            proj = {}
            for n in args.cfg4_project:
                b = cfg4_block(args, 1, 0, dev, barrier, shard_world=n)
                proj[str(n)] = {"streams_per_gpu": b["streams_per_rank"], "per_gpu_frames_per_s": b["frames_per_s"],
                                "ms_per_step": b["ms_per_step"],
                                "projected_total_frames_per_s": b["frames_per_s"] * n,
                                "projected_scaling_vs_1": b["frames_per_s"] * n / c4["frames_per_s"]}
            c4["per_gpu_share_at_n_gpus"] = proj

    if rank == 0:
        summ = summarize(per_rank)
        value = summ["frames_per_s"]
        e2e_value = summarize(e2e_all)["frames_per_s"] if e2e_ms else None
        max_ms = summ["max_elapsed_ms"]
        peak, peak_kind = peaks()
        nfr = K * F
        kpf, rpf, cpf = kept / nfr, recs / nfr, cand / nfr
        # SURVEY 8(d) algorithmic bytes of the timed frames
        byt = alg_bytes(nfr, esz, cand, kept, recs)
        assoc_launch_ms = as_ms.value / max(nup.value, 1)
        frame_launch_ms = fr_ms.value / max(nup.value, 1)
        dominant = "associate_kernel" if as_ms.value >= fr_ms.value else "frame_heads_kernel"
        dom_ms = assoc_launch_ms if dominant == "associate_kernel" else frame_launch_ms
        bytes_launch = byt / K
        achieved = bytes_launch / (dom_ms / 1e3) / 1e9
        step_gbs = byt / (ms / 1e3) / 1e9
        # the kernels' own input/output bytes (diagnostics, per launch)
        assoc_own = F * (4 * D * kpf + 2 * 4 * D * kpf + 48 * rpf + 40 * kpf)
        frame_own = F * (8 * esz * N_CELLS + cpf * esz * (4 + D) + 4 * D * kpf + 40 * kpf)
        traffic = None
        tfile = ROOT / "profiles" / "traffic.json"
        if tfile.exists():
            traffic = json.loads(tfile.read_text()).get(args.config, {}).get(dominant)
        run = {"generation": "streamed between steps, steps timed one by one" if streamed
               else "pre-generated on device", "pipeline": "decode of step i+1 overlaps association of step i"
               if pipe else "off", "parallelism": f"streams sharded over {world} rank(s), final NCCL all_gather",
               "streams_per_rank": S}
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": max_ms / K, "higher_is_better": True, "scaling": "strong" if multi else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world), "run": run,
            "e2e": {"value": e2e_value, "unit": "frames/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "steps": e2e_steps if e2e_ms else 0,
                    "kernels": e2e_kernels, **({"unavailable": e2e_reason} if e2e_reason else {})},
            "roofline": {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_launch": bytes_launch, "ms_per_launch": dom_ms,
                         "bytes_def": "SURVEY 8(d): per frame 8*4*N_cells + 16*C + 4*D*K + 48*R with this run's "
                                      "C, K, R (fp32; input terms halve for fp16 inputs)",
                         "step": {"achieved": step_gbs, "frac": step_gbs / peak},
                         "note": "association is a per-stream dependency chain (latency-bound); DESIGN.md s6"},
            "kernels": {
                "event_sample_stride": prof_stride,
                "frame_heads_kernel": {"ms_per_launch": frame_launch_ms, "own_bytes_per_launch": frame_own,
                                       "own_GBps": frame_own / (frame_launch_ms / 1e3) / 1e9},
                "associate_kernel": {"ms_per_launch": assoc_launch_ms, "own_bytes_per_launch": assoc_own,
                                     "own_GBps": assoc_own / (assoc_launch_ms / 1e3) / 1e9,
                                     "share_of_step": as_ms.value / max(ms, 1e-9)}},
            "per_frame": {"candidates": cpf, "detections": kpf, "records": rpf},
            "parity": parity,
            "cfg4": c4,
            "assoc_phases_us_per_frame": {
                name: float(phase[i]) / max(phase[11], 1) / (clocks.summary()["sm_mhz"] or 1965)
                for i, name in list(enumerate(["load_predict", "gate", "csr", "cost", "lap", "match",
                                               "update_ema", "records_births"]))
                + [(16, "lap.components_tiecheck"), (17, "lap.peeling"), (18, "lap.residual_setup"),
                   (19, "lap.warp_solves"), (20, "lap.full_restatement"), (31, "whole_frame"),
                   (28, "launch.prologue"), (29, "launch.epilogue")]},
            "assoc_counters_per_frame": {name: float(phase[i]) / max(phase[11], 1) for i, name in
                                         [(8, "tie_fallback"), (9, "finite_entries"), (10, "multi_components"),
                                          (14, "residual_entries"), (12, "tracks"), (13, "detections"),
                                          (15, "peel_rounds")]},
            "ranks": per_rank,
            "gpu_launches": n_launch,
            "clocks": clocks.summary(),
            "quality": quality,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def timed_updates_host(bt, host_batches, hout, stream):
    import torch

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for hb in host_batches:
        bt.update(hb, host_out=hout, sync=False)
    bt.join()                      # ... and after the last records reached host memory
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg1", choices=["cfg0", "cfg1", "cfg2", "cfg3", "cfg4"])
    ap.add_argument("--batch", type=int, default=None, help="frames per stream per update (default: config's B)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--e2e-host-gb", type=float, default=24.0)
    ap.add_argument("--cpu-stream-frames", type=int, default=100)
    ap.add_argument("--ref-budget-s", type=float, default=30.0)
    ap.add_argument("--cfg4-steps", type=int, default=4)
    ap.add_argument("--cfg4-warmup", type=int, default=3)
    ap.add_argument("--no-cfg4", action="store_true", help="skip the config-4 strong-scaling block")
    ap.add_argument("--cfg4-project", type=int, nargs="*", default=[8],
                    help="N=1 only: also time rank 0's cfg4 shard at these GPU counts (per-GPU work at N GPUs)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-pipeline", action="store_true", help="serialise decode and association")
    ap.add_argument("--jde", action="store_true",
                    help="JDE extensions on (lambda = 0.98 fused cost, IoU second stage at 0.5); off = reference path")
    ap.add_argument("--dtype", default="f32", choices=["f32", "f16"],
                    help="head / embedding input type (f16 = MIXED-precision input mode, SURVEY 8(f))")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = os.environ.get("WORLD_SIZE")
    if world is None and args.gpus > 1:
        # one process per GPU: re-launch under torchrun (NCCL, 127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
               *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    if world is not None and int(world) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
