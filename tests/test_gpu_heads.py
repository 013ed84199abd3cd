"""GPU parity of the batched update(head_outputs) path against the CPU oracle.

Inputs are generated on the device, copied back, and decoded + tracked by the
oracle (oracle/heads.py + oracle/tracker.py). Bit-exact: kept detection
indices (global anchor codes), association pairs (detection -> track id),
record ids. Values: boxes, objectness, match costs within 1e-4 relative
(the north-star tolerance; observed errors are reported and are ~1e-15).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from oracle import tracker as ot   # noqa: E402
from parity import FrameCompare, host_frames, oracle_settings, run_oracle_frame   # noqa: E402


def _pkg():
    import paper_2011_03910_b200 as p
    from paper_2011_03910_b200 import synth
    return p, synth


def _launch_info(bt):
    import ctypes as C
    th, cl = C.c_int32(), C.c_int32()
    bt.engine.lib.tf_launch_info(bt.engine.ctx, C.byref(th), C.byref(cl))
    return th.value, cl.value


def _run_parity(cfg_name, steps, B, streams=1, quantize=False, literal=False, config=None, max_tracks=256,
                half=False, max_detections=256, expect_threads=None, check_streams=None, max_candidates=512,
                **synth_kw):
    """GPU update of `streams` streams x B frames per step against one oracle
    tracker per checked stream (all streams by default; full-size configs
    check a sample, the other streams still run on the GPU in the same
    launches)."""
    p, synth = _pkg()
    cfg = config or p.TrackerConfig()
    gen = synth.make(cfg_name, device="cuda", streams=streams, literal_noise=literal, **synth_kw)
    cap = p.Capacity(streams=streams, max_frames=streams * B, max_tracks=max_tracks, max_detections=max_detections,
                     max_candidates=max_candidates)
    bt = p.BatchTracker(streams, cfg, frames_per_update=B, quantize=quantize, capacity=cap)
    if expect_threads is not None:
        assert _launch_info(bt)[0] == expect_threads
    checked = list(range(streams)) if check_streams is None else list(check_streams)
    oracles = {s: ot.OracleTracker(oracle_settings(cfg, quantize)) for s in checked}
    cmp = FrameCompare()
    frame = 0
    for step in range(steps):
        out = gen.next_batch(B)
        if half:
            out = out.half()
        fidx = np.array([[frame + b for b in range(B)] for _ in range(streams)], np.int64)
        res = bt.update(out, fidx, trace=True)
        tr = {k: v.cpu().numpy() for k, v in bt.trace(streams * B).items()}
        cnt = res.count.cpu().numpy()
        ids, boxes, objs = res.track_id.cpu().numpy(), res.box.cpu().numpy(), res.objectness.cpu().numpy()
        sel = [s * B + b for s in checked for b in range(B)]
        host = dict(zip(sel, host_frames(out, sel)))
        for s in checked:
            for b in range(B):
                f = s * B + b
                codes, trace = run_oracle_frame(oracles[s], frame + b, *host[f], quantize=quantize)
                assert tr["cand_count"][f] == len(codes), f"candidate count differs at frame {f}"
                k = tr["det_count"][f]
                recs = [(int(ids[f, i]), tuple(boxes[f, i]), float(objs[f, i])) for i in range(cnt[f])]
                cmp.check(frame + b, trace, recs, tr["det_code"][f, :k], tr["det_track"][f, :k],
                          tr["det_cost"][f, :k], tr["det_matched"][f, :k], codes)
        del out, host
        frame += B
    # final track tables
    for s in checked:
        ex = bt.export(s)
        o = oracles[s]
        assert ex["track_id"].tolist() == [t.track_id for t in o.tracks]
        assert ex["hits"].tolist() == [t.hits for t in o.tracks]
        assert [int(v) for v in ex["state"]] == [int(t.state == ot.LOST) for t in o.tracks]
        for i, t in enumerate(o.tracks):
            np.testing.assert_allclose(ex["mean"][i], t.mean, rtol=1e-4, atol=1e-6)
            np.testing.assert_allclose(ex["covariance"][i], t.cov, rtol=1e-4, atol=1e-9)
            np.testing.assert_allclose(ex["embedding"][i], t.emb, rtol=1e-4, atol=1e-6)
        assert ex["next_id"] == o.next_id
    return cmp


def test_cfg0_single_stream_b1():
    cmp = _run_parity("cfg0", steps=40, B=1)
    assert cmp.matches > 500
    print(f"cfg0: frames={cmp.frames} records={cmp.records} matches={cmp.matches} "
          f"box_rel={cmp.max_box_rel:.2e} cost_rel={cmp.max_cost_rel:.2e}")


def test_cfg1_batch32():
    cmp = _run_parity("cfg1", steps=3, B=32)
    print(f"cfg1/B32: frames={cmp.frames} records={cmp.records} matches={cmp.matches} "
          f"box_rel={cmp.max_box_rel:.2e} cost_rel={cmp.max_cost_rel:.2e}")


def test_multi_stream_cfg3_like():
    cmp = _run_parity("cfg3", steps=3, B=8, streams=6)
    assert cmp.frames == 6 * 24


def test_dense_scene_cfg2_like():
    # 512 tracks: the association CTA keeps fewer entries on chip, so frames
    # alternate between on-chip and pooled (global) entry storage
    cmp = _run_parity("cfg2", steps=3, B=8, max_tracks=512)
    assert cmp.records > 1000


def test_mixed_precision_quantize():
    _run_parity("cfg0", steps=12, B=2, quantize=True)


def test_literal_noise_stress():
    _run_parity("cfg0", steps=10, B=2, literal=True, max_tracks=512)


def test_euclidean_and_lifecycle_knobs():
    p, _ = _pkg()
    cfg = p.TrackerConfig(gate_metric="euclidean", gate_threshold=2500.0, max_lost=3, min_hits=2)
    _run_parity("cfg0", steps=10, B=3, config=cfg)


def test_host_pinned_input_matches_device_input():
    p, synth = _pkg()
    gen = synth.make("cfg1", device="cuda")
    out = gen.next_batch(8)
    dev = p.BatchTracker(1, frames_per_update=8)
    host = p.BatchTracker(1, frames_per_update=8)
    r1 = dev.update(out)
    pinned = p.HeadOutputs(tuple(h.cpu().pin_memory() for h in out.heads),
                           tuple(e.cpu().pin_memory() for e in out.embs))
    # keep channels_last on the host copy so the gather stays contiguous
    pinned = p.HeadOutputs(pinned.heads, tuple(e.contiguous(memory_format=torch.channels_last).pin_memory()
                                               for e in pinned.embs))
    r2 = host.update(pinned)
    assert np.array_equal(r1.count.cpu().numpy(), r2.count.numpy())
    for f in range(8):
        n = int(r2.count[f])
        assert np.array_equal(r1.track_id[f, :n].cpu().numpy(), r2.track_id[f, :n].numpy())
        assert np.array_equal(r1.box[f, :n].cpu().numpy(), r2.box[f, :n].numpy())


def test_ordering_error_and_capacity():
    p, synth = _pkg()
    gen = synth.make("cfg0", device="cuda")
    bt = p.BatchTracker(1, frames_per_update=2)
    bt.update(gen.next_batch(2), np.array([5, 6]))
    with pytest.raises(p.OrderingError):
        bt.update(gen.next_batch(2), np.array([6, 7]))
    small = p.BatchTracker(1, frames_per_update=1, capacity=p.Capacity(streams=1, max_frames=1,
                                                                           max_candidates=8))
    with pytest.raises(p.CapacityError):
        small.update(gen.next_batch(1))


def test_full_size_cfg4_step_properties():
    """One cfg4-sized step (512 streams x 8 frames): size-independent invariants."""
    p, synth = _pkg()
    gen = synth.make("cfg4", device="cuda", streams=512)
    bt = p.BatchTracker(512, frames_per_update=8)
    last_max = np.zeros(512, np.int64)
    for _ in range(2):
        res = bt.update(gen.next_batch(8), trace=True)
        cnt = res.count.cpu().numpy()
        ids = res.track_id.cpu().numpy()
        tr = bt.trace(512 * 8)
        det = tr["det_count"].cpu().numpy()
        assert np.array_equal(cnt, det)              # min_hits = 1: every kept detection is reported
        for f in range(512 * 8):
            row = ids[f, :cnt[f]]
            assert np.all(np.diff(row) > 0)          # sorted by id, unique
        for s in range(512):
            blk = ids[s * 8:(s + 1) * 8]
            m = blk.max() if blk.size else 0
            assert m >= last_max[s]
            last_max[s] = m


def test_cluster_and_single_cta_association_agree(monkeypatch):
    """The cluster-cooperative association (followers compute costs / EMA via
    DSMEM) and the single-CTA path produce identical records and traces."""
    p, synth = _pkg()
    outs = []
    for cl in ("1", "8"):
        monkeypatch.setenv("TF_CLUSTER", cl)
        gen = synth.make("cfg1", device="cuda", seed=11)
        bt = p.BatchTracker(1, frames_per_update=16)
        res = []
        for _ in range(3):
            r = bt.update(gen.next_batch(16), trace=True)
            tr = bt.trace(16)
            res.append((r.count.cpu().numpy().copy(), r.track_id.cpu().numpy().copy(), r.box.cpu().numpy().copy(),
                        tr["det_cost"].cpu().numpy().copy()))
        outs.append(res)
    for (c1, i1, b1, k1), (c8, i8, b8, k8) in zip(*outs):
        assert np.array_equal(c1, c8)
        for f in range(16):
            n = c1[f]
            assert np.array_equal(i1[f, :n], i8[f, :n])
            assert np.array_equal(b1[f, :n], b8[f, :n])
            assert np.array_equal(np.nan_to_num(k1[f, :n]), np.nan_to_num(k8[f, :n]))


def test_narrow_association_ctas_match_oracle(monkeypatch):
    """The 128-thread association CTAs (two per SM, chosen for launches with
    more streams than twice the SM count) against the oracle, forced on a
    small cfg3-like launch."""
    monkeypatch.setenv("TF_ASSOC_NARROW", "1")
    cmp = _run_parity("cfg3", steps=3, B=8, streams=6, max_tracks=192, max_detections=128, expect_threads=128)
    assert cmp.frames == 6 * 24


def test_overlapped_decode_and_association_match_oracle(monkeypatch):
    """Opt-in overlapped mode (TF_OVERLAP): a persistent decode grid publishes
    frames through per-frame ready flags and the association, launched as its
    programmatic dependent, waits per frame instead of on the grid. 40 streams
    x 8 frames (>= 2 x SMs frames) with 128-thread association CTAs, 3 steps,
    four streams checked against the oracle."""
    monkeypatch.setenv("TF_ASSOC_NARROW", "1")
    monkeypatch.setenv("TF_OVERLAP", "1")
    cmp = _run_parity("cfg4", steps=3, B=8, streams=40, check_streams=[0, 13, 27, 39], max_candidates=192,
                      max_detections=96, max_tracks=160, expect_threads=128)
    assert cmp.frames == 4 * 24


@pytest.mark.parametrize("cluster,narrow", [("16", False), ("1", False), ("1", True)])
def test_pooled_entries_path_matches_oracle(monkeypatch, cluster, narrow):
    """Frames whose gated entries exceed the on-chip capacity keep them in the
    stream's global pool; forced here with a tiny capacity, for the cluster,
    single-CTA and 128-thread associations."""
    monkeypatch.setenv("TF_CAP_ENTRIES", "64")
    monkeypatch.setenv("TF_CLUSTER", cluster)
    if narrow:
        monkeypatch.setenv("TF_ASSOC_NARROW", "1")
    cmp = _run_parity("cfg1", steps=2, B=8, max_tracks=160, max_detections=96,
                      expect_threads=128 if narrow else 256)
    assert cmp.frames == 16


def test_narrow_and_wide_association_agree(monkeypatch):
    """128- and 256-thread association CTAs give identical records and traces."""
    p, synth = _pkg()
    outs = []
    for env in ("TF_ASSOC_NARROW", "TF_ASSOC_WIDE"):
        monkeypatch.delenv("TF_ASSOC_NARROW", raising=False)
        monkeypatch.delenv("TF_ASSOC_WIDE", raising=False)
        monkeypatch.setenv(env, "1")
        gen = synth.make("cfg4", device="cuda", streams=16, seed=5)
        cap = p.Capacity(streams=16, max_frames=16 * 8, max_candidates=192, max_detections=96, max_tracks=160)
        bt = p.BatchTracker(16, frames_per_update=8, capacity=cap)
        assert _launch_info(bt)[0] == (128 if env == "TF_ASSOC_NARROW" else 256)
        res = []
        for _ in range(3):
            r = bt.update(gen.next_batch(8), trace=True)
            tr = bt.trace(16 * 8)
            res.append((r.count.cpu().numpy().copy(), r.track_id.cpu().numpy().copy(), r.box.cpu().numpy().copy(),
                        tr["det_cost"].cpu().numpy().copy()))
        outs.append(res)
    for (c1, i1, b1, k1), (c2, i2, b2, k2) in zip(*outs):
        assert np.array_equal(c1, c2)
        for f in range(16 * 8):
            n = c1[f]
            assert np.array_equal(i1[f, :n], i2[f, :n])
            assert np.array_equal(b1[f, :n], b2[f, :n])
            assert np.array_equal(np.nan_to_num(k1[f, :n]), np.nan_to_num(k2[f, :n]))


def test_longest_first_order_does_not_change_results(monkeypatch):
    """More single-CTA streams than resident association slots: from the
    second update on, blocks take streams in longest-first order (lpt_order).
    Records, costs and the final track tables are bit-identical to the
    identity order (TF_NO_LPT)."""
    import torch

    p, synth = _pkg()
    S, B = 2 * torch.cuda.get_device_properties(0).multi_processor_count + 24, 2
    outs = []
    for no_lpt in (False, True):
        monkeypatch.delenv("TF_NO_LPT", raising=False)
        if no_lpt:
            monkeypatch.setenv("TF_NO_LPT", "1")
        gen = synth.make("cfg4", device="cuda", streams=S, seed=11)
        cap = p.Capacity(streams=S, max_frames=S * B, max_candidates=192, max_detections=96, max_tracks=160)
        bt = p.BatchTracker(S, frames_per_update=B, capacity=cap)
        assert _launch_info(bt)[0] == 128
        res = []
        for _ in range(3):
            b = gen.next_batch(B)
            r = bt.update(b, trace=True)
            tr = bt.trace(S * B)
            res.append((r.count.cpu().numpy().copy(), r.track_id.cpu().numpy().copy(), r.box.cpu().numpy().copy(),
                        tr["det_cost"].cpu().numpy().copy()))
            del b
        res.append([bt.export(s) for s in (0, S // 2, S - 1)])
        outs.append(res)
        del bt, gen
        torch.cuda.empty_cache()
    for (c1, i1, b1, k1), (c2, i2, b2, k2) in zip(outs[0][:3], outs[1][:3]):
        assert np.array_equal(c1, c2)
        assert np.array_equal(i1, i2) and np.array_equal(b1, b2)
        assert np.array_equal(np.nan_to_num(k1), np.nan_to_num(k2))
    for e1, e2 in zip(outs[0][3], outs[1][3]):
        assert all(np.asarray(e1[k]).tobytes() == np.asarray(e2[k]).tobytes() for k in e1)


def test_stream_hold_releases():
    """tf_stream_hold: work queued behind the hold runs only after the host
    releases the pinned flag (bench.py's single-update timing)."""
    import time

    import torch
    from paper_2011_03910_b200 import _lib

    lib = _lib.load()
    flag = torch.zeros(1, dtype=torch.int32).pin_memory()
    x = torch.zeros(1, device="cuda")
    st = torch.cuda.current_stream()
    assert lib.tf_stream_hold(flag.data_ptr(), st.cuda_stream) == 0
    x += 1
    done = torch.cuda.Event()
    done.record(st)
    time.sleep(0.05)
    assert not done.query()              # still held
    flag.fill_(1)
    done.synchronize()
    assert float(x.item()) == 1.0


def _run_ext(cfg_name, config, **kw):
    """_run_parity, also returning the oracle's IoU-stage match count."""
    import oracle.tracker as ot
    counts = []
    orig = ot.OracleTracker.__init__

    def init(self, settings=None):
        orig(self, settings)
        counts.append(self)
    ot.OracleTracker.__init__ = init
    try:
        cmp = _run_parity(cfg_name, config=config, **kw)
    finally:
        ot.OracleTracker.__init__ = orig
    return cmp, sum(o.stage2_matches for o in counts)


def test_jde_extensions_match_oracle():
    """lambda-fused cost + IoU second stage (JDE extensions, off on the
    reference path) against the oracle's restatement of them."""
    p, _ = _pkg()
    cfg = p.TrackerConfig(motion_lambda=0.98, iou_stage=True, iou_threshold=0.5)
    cmp, _ = _run_ext("cfg1", cfg, steps=4, B=8)
    assert cmp.frames == 32 and cmp.matches > 0


def test_iou_stage_takes_over_dissolved_matches():
    """A strict cosine threshold dissolves most first-stage matches; the IoU
    stage re-associates them, exactly as the oracle does."""
    p, _ = _pkg()
    cfg = p.TrackerConfig(max_cost=0.02, motion_lambda=0.98, iou_stage=True, iou_threshold=0.5)
    cmp, n2 = _run_ext("cfg1", cfg, steps=3, B=8)
    assert n2 > 50, n2
    cmp, n2 = _run_ext("cfg3", cfg, steps=2, B=8, streams=6)
    assert n2 > 20, n2


def test_pipelined_updates_match_serial():
    """Pipelining (decode of update i+1 overlapping association of update i on
    a side stream, double-buffered detections) gives the serial results."""
    p, synth = _pkg()
    res = []
    for pipe in (False, True):
        gen = synth.make("cfg1", device="cuda", seed=5)
        batches = [gen.next_batch(8) for _ in range(4)]
        bt = p.BatchTracker(1, frames_per_update=8, pipeline=pipe)
        hout = [bt.host_output(8) for _ in batches] if pipe else None
        outs = []
        for i, bb in enumerate(batches):
            if pipe:
                pinned = p.HeadOutputs(tuple(h.cpu().pin_memory() for h in bb.heads),
                                       tuple(e.cpu().pin_memory() for e in bb.embs))
                r = bt.update(pinned, host_out=hout[i], sync=False)
                outs.append(r)                       # distinct pinned buffers per update
            else:
                r = bt.update(bb)
                outs.append((r.count.cpu().numpy().copy(), r.track_id.cpu().numpy().copy()))
        bt.finish()
        if pipe:
            outs = [(o.count.numpy().copy(), o.track_id.numpy().copy()) for o in outs]
        res.append(outs)
    for (c0, i0), (c1, i1) in zip(*res):
        assert np.array_equal(np.asarray(c0), np.asarray(c1))
        for f in range(8):
            n = int(c0[f])
            assert np.array_equal(i0[f, :n], i1[f, :n])


def test_native_fp16_inputs():
    """MIXED-precision input mode: binary16 head tensors
    and embedding maps are read natively (half the input bytes). Every fp16
    value is exact in fp32/fp64, so the oracle decodes the same fp16 arrays
    and the decisions must stay bit-exact."""
    cmp = _run_parity("cfg1", steps=2, B=16, half=True)
    assert cmp.matches > 500
    cmp = _run_parity("cfg0", steps=10, B=4, half=True, quantize=True)
    assert cmp.matches > 100


def test_fp16_layout_errors():
    p, synth = _pkg()
    gen = synth.make("cfg0", device="cuda")
    out = gen.next_batch(2)
    mixed = p.HeadOutputs(tuple(h.half() for h in out.heads), out.embs)   # fp16 heads, fp32 maps
    bt = p.BatchTracker(1, frames_per_update=2)
    with pytest.raises(p.LayoutError):
        bt.update(mixed)


def test_profiling_event_stride():
    """tf_set_profiling(level | stride << 4) records kernel events on every
    stride-th update only (bench.py samples them at small batches)."""
    import ctypes as C
    p, synth = _pkg()
    gen = synth.make("cfg0", device="cuda", seed=3)
    bt = p.BatchTracker(1, frames_per_update=1)
    lib = bt.engine.lib
    lib.tf_set_profiling(bt.engine.ctx, 1 | (4 << 4))
    for _ in range(8):
        bt.update(gen.next_batch(1), sync=False)
    bt.join()
    fr, asc, n = C.c_double(), C.c_double(), C.c_int64()
    lib.tf_kernel_times(bt.engine.ctx, C.byref(fr), C.byref(asc), C.byref(n))
    lib.tf_set_profiling(bt.engine.ctx, 0)
    assert n.value == 2 and fr.value > 0 and asc.value > 0
    assert _launch_info(bt)[0] == 256


# ---------------------------------------------------------------- full-size shapes, sampled streams
def test_full_cfg3_sampled_streams_match_oracle():
    """BASELINE config 3 at its bench shape (64 streams x B = 8, 10-100
    objects per stream): every stream runs in the same launches, four are
    checked against the oracle over three updates."""
    cmp = _run_parity("cfg3", steps=3, B=8, streams=64, check_streams=[0, 21, 42, 63], max_candidates=256,
                      max_detections=160)
    assert cmp.frames == 4 * 24 and cmp.matches > 1000


def test_full_cfg4_sampled_streams_match_oracle():
    """BASELINE config 4 at its 1-GPU bench shape (512 streams x B = 8, the
    bench's capacities): streams 0, 137, 300 and 511 against the oracle over
    three updates."""
    cmp = _run_parity("cfg4", steps=3, B=8, streams=512, check_streams=[0, 137, 300, 511], max_candidates=192,
                      max_detections=96, max_tracks=160, expect_threads=128)   # two association CTAs per SM
    assert cmp.frames == 4 * 24 and cmp.matches > 3000


# ---------------------------------------------------------------- determinism
def _replay(batches, streams, B, **kw):
    p, _ = _pkg()
    cap = p.Capacity(streams=streams, max_frames=streams * B, **kw)
    bt = p.BatchTracker(streams, frames_per_update=B, capacity=cap)
    outs = []
    for out in batches:
        r = bt.update(out, trace=True)
        tr = bt.trace(streams * B)
        outs.append([t.cpu().numpy().copy() for t in (r.count, r.track_id, r.box, r.objectness, tr["cand_count"],
                                                      tr["det_count"], tr["det_code"], tr["det_track"],
                                                      tr["det_cost"], tr["det_matched"])])
    ex = [bt.export(s) for s in range(streams)]
    return outs, ex


@pytest.mark.parametrize("cfg_name,streams,B", [("cfg1", 1, 32), ("cfg3", 16, 8), ("cfg2", 1, 8), ("cfg4", 512, 8)])
def test_deterministic_replay(cfg_name, streams, B):
    """Run the default variant twice on identical inputs: every output, trace
    and final track table is bit-identical (race
    detection by deterministic replay)."""
    _, synth = _pkg()
    gen = synth.make(cfg_name, device="cuda", streams=streams, seed=23)
    if cfg_name == "cfg4":               # one 119 GB batch fits, fed twice (frame indices advance)
        b0 = gen.next_batch(B)
        batches = [b0, b0]
    else:
        batches = [gen.next_batch(B) for _ in range(3)]
    kw = {"cfg2": dict(max_tracks=384, max_candidates=768, max_detections=224),
          "cfg4": dict(max_tracks=160, max_candidates=192, max_detections=96)}.get(cfg_name, {})
    a, ea = _replay(batches, streams, B, **kw)
    b, eb = _replay(batches, streams, B, **kw)
    for step_a, step_b in zip(a, b):
        for x, y in zip(step_a, step_b):
            assert x.tobytes() == y.tobytes()
    for x, y in zip(ea, eb):
        for k in x:
            assert np.asarray(x[k]).tobytes() == np.asarray(y[k]).tobytes(), k


# ---------------------------------------------------------------- boundary: embedding map width / device
def test_embedding_map_width_mismatch_is_layout_error():
    """parse_output rejects rows whose width is not 6 + embedding_dim
    (tf/postproc.py:25-29); a narrower (or wider) embedding map is the same
    mistake here and must raise LayoutError, never gather neighbouring cells."""
    p, synth = _pkg()
    gen = synth.make("cfg0", device="cuda", dim=64)
    out = gen.next_batch(2)
    bt = p.BatchTracker(1, p.TrackerConfig(embedding_dim=128), frames_per_update=2)
    with pytest.raises(p.LayoutError, match="channels"):
        bt.update(out)
    ok = p.BatchTracker(1, p.TrackerConfig(embedding_dim=64), frames_per_update=2)
    ok.update(out)


def test_embedding_map_on_another_device_is_layout_error():
    p, synth = _pkg()
    gen = synth.make("cfg0", device="cuda")
    out = gen.next_batch(1)
    mixed = p.HeadOutputs(out.heads, (out.embs[0].cpu(),) + tuple(out.embs[1:]))
    bt = p.BatchTracker(1, frames_per_update=1)
    with pytest.raises(p.LayoutError):
        bt.update(mixed)


def test_c_abi_rejects_channel_count_mismatch():
    """The C side checks tf_head_scale.channels against embedding_dim itself
    (a caller that bypasses the Python shim gets TF_LAYOUT, not a silent
    out-of-bounds gather)."""
    import ctypes as C
    p, synth = _pkg()
    from paper_2011_03910_b200 import _lib
    from paper_2011_03910_b200.heads import heads_descriptor
    gen = synth.make("cfg0", device="cuda")
    out = gen.next_batch(1)
    bt = p.BatchTracker(1, frames_per_update=1)
    desc = heads_descriptor(out, False, 512)
    desc.scale[1].channels = 511
    eng = bt.engine
    code = eng.lib.tf_update_heads(eng.ctx, C.byref(desc), 0, 1, 1, np.zeros(1, np.int64).ctypes.data,
                                   C.byref(eng.records), None, _lib.stream_handle())
    assert code == 6 and b"511" in eng.lib.tf_last_error(eng.ctx)


# ---------------------------------------------------------------- decode pinned to the generator's truth
def test_gpu_decode_reproduces_generator_boxes():
    """Independent pin of the decode (the reference has none): with zero
    box-delta noise the generator encodes each visible object's true box at
    its anchor cell; on the first frame every track is a birth whose
    posterior box is its measurement, so the GPU records must reproduce the
    truth boxes (1e-6 relative; objects whose centre fraction hit the
    generator's 1e-3 clamp are excluded)."""
    import torch as T
    p, synth = _pkg()
    from decode_pin import match_truth
    for seed in range(3):
        gen = synth.make("cfg1", device="cuda", seed=seed, delta_sigma=0.0)
        gen.record_truth()
        out = gen.next_batch(1)
        bt = p.BatchTracker(1, frames_per_update=1)
        res = bt.update(out)
        n = int(res.count[0])
        boxes = res.box[0, :n].cpu().numpy()
        obj = res.objectness[0, :n].cpu().numpy()
        true_obj = np.isclose(obj, 1.0 / (1.0 + np.exp(-8.0)), rtol=1e-12, atol=0.0)   # the +4 / -4 logits
        _, _, _, truth = gen.truth[0]
        active = gen.active[0].cpu().numpy()
        checked = match_truth(boxes[true_obj], truth[0].cpu().numpy()[active], rtol=1e-6)
        assert checked >= 40, checked
        del out
        T.cuda.empty_cache()
