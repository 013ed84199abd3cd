"""Seeded synthetic JDE head tensors for BASELINE.json configs 0-4.

Stands in for the network forward (the reference likewise replaces the JDE
model with a seeded synthetic source, tf/detgen.py:1-16, and emits
already-decoded rows; this generator emits the *head tensors* instead, so the
decode is exercised). Generation runs on the target device with torch and is
never inside a timed region.

Decisions:
* 1920x1080 frames letterboxed to 1088x608 (scale 608/1080, pad_x 3.5);
* each visible object is encoded at its best wh-IoU anchor among the 12, at
  cell floor(centre / stride): deltas t = logit(clamp(frac, 1e-3, 1 - 1e-3)),
  ln(size / anchor), plus N(0, 0.05); background logit -4, foreground +4;
  later objects overwrite earlier ones on a collision (deterministically);
* every other anchor: background logit 0, foreground ~ N(-4, 1) (~1.7 spurious
  candidates per frame), deltas ~ N(0, 1); embeddings ~ N(0, 1/D) per dim;
* identity embeddings are random unit vectors; per-frame noise is per-vector
  sigma 0.1 (per-dim 0.1/sqrt(D)); ``literal_noise`` uses per-dim sigma 0.1;
* velocities N(0, 3) px/frame per axis (config 2: directed toward the frame
  centre); heights U(40, 300), aspect w/h 0.41; 5% occlusion dropout (20% for
  config 2); an object leaving the frame respawns as a new identity at a
  uniform position with a fresh velocity, so N objects stay in view.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import torch

from .heads import ANCHORS, GRID, HeadOutputs, IMAGE_H, IMAGE_W, STRIDES, letterbox


@dataclass(frozen=True)
class SynthConfig:
    streams: int = 1
    objects: tuple[int, int] = (50, 50)     # per stream, uniform in [lo, hi]
    frames: int = 100                        # per stream
    batch: int = 1                           # frames per stream per update (B)
    p_miss: float = 0.05
    emb_sigma: float = 0.1
    literal_noise: bool = False
    delta_sigma: float = 0.05
    height_range: tuple[float, float] = (40.0, 300.0)
    aspect: float = 0.41
    vel_sigma: float = 3.0
    toward_center: bool = False
    dim: int = 512
    seed: int = 0


CONFIGS = {
    "cfg0": SynthConfig(streams=1, objects=(20, 20), frames=100, batch=1),
    "cfg1": SynthConfig(streams=1, objects=(50, 50), frames=1000, batch=32),
    "cfg2": SynthConfig(streams=1, objects=(200, 200), frames=300, batch=8, p_miss=0.2, toward_center=True),
    "cfg3": SynthConfig(streams=64, objects=(10, 100), frames=500, batch=8),
    "cfg4": SynthConfig(streams=512, objects=(50, 50), frames=1000, batch=8),
}


def _anchor_table(device):
    """12 anchors in (scale index in STRIDES order, anchor) order, input pixels."""
    rows = []
    for si, s in enumerate(STRIDES):
        for a, (aw, ah) in enumerate(ANCHORS[s]):
            rows.append((si, a, aw, ah))
    t = torch.tensor(rows, dtype=torch.float64, device=device)
    return t[:, 0].long(), t[:, 1].long(), t[:, 2], t[:, 3]


class HeadSynth:
    """Stateful generator: each call to :meth:`next_batch` advances every
    stream by ``B`` frames and returns their head tensors (stream-major)."""

    def __init__(self, cfg: SynthConfig, device="cuda"):
        self.cfg = cfg
        self.device = torch.device(device)
        self.gen = torch.Generator(device=self.device)
        self.gen.manual_seed(int(cfg.seed))
        S = cfg.streams
        lo, hi = cfg.objects
        self.nmax = hi
        counts = torch.randint(lo, hi + 1, (S,), generator=self.gen, device=self.device)
        self.active = torch.arange(hi, device=self.device)[None, :] < counts[:, None]     # [S, N]
        self.scale_inv, self.pad_x, self.pad_y = letterbox()
        self.r = 1.0 / self.scale_inv
        self.frame = 0
        self.next_identity = 1
        self.truth = None          # list of per-frame ground truth once record_truth() was called
        shape = (S, hi)
        self.cx = torch.zeros(shape, dtype=torch.float64, device=self.device)
        self.cy = torch.zeros_like(self.cx)
        self.vx = torch.zeros_like(self.cx)
        self.vy = torch.zeros_like(self.cx)
        self.h = torch.zeros_like(self.cx)
        self.ident = torch.zeros(S, hi, cfg.dim, dtype=torch.float32, device=self.device)
        self.gid = torch.zeros(shape, dtype=torch.int64, device=self.device)   # ground-truth identity
        self._respawn(torch.ones(shape, dtype=torch.bool, device=self.device))
        self.an_si, self.an_a, self.an_w, self.an_h = _anchor_table(self.device)

    # ---------------------------------------------------------------------
    def _rand(self, *shape, dtype=torch.float64):
        return torch.rand(*shape, generator=self.gen, device=self.device, dtype=dtype)

    def _randn(self, *shape, dtype=torch.float64):
        return torch.randn(*shape, generator=self.gen, device=self.device, dtype=dtype)

    def _respawn(self, mask):
        c = self.cfg
        S, N = mask.shape
        h = c.height_range[0] + (c.height_range[1] - c.height_range[0]) * self._rand(S, N)
        cx = IMAGE_W * self._rand(S, N)
        cy = IMAGE_H * self._rand(S, N)
        if c.toward_center:
            speed = self._randn(S, N).abs() * c.vel_sigma
            dx, dy = IMAGE_W / 2.0 - cx, IMAGE_H / 2.0 - cy
            norm = torch.sqrt(dx * dx + dy * dy).clamp_min(1e-6)
            vx, vy = speed * dx / norm, speed * dy / norm
        else:
            vx, vy = c.vel_sigma * self._randn(S, N), c.vel_sigma * self._randn(S, N)
        e = self._randn(S, N, c.dim, dtype=torch.float32)
        e = e / e.norm(dim=2, keepdim=True)
        self.cx = torch.where(mask, cx, self.cx)
        self.cy = torch.where(mask, cy, self.cy)
        self.vx = torch.where(mask, vx, self.vx)
        self.vy = torch.where(mask, vy, self.vy)
        self.h = torch.where(mask, h, self.h)
        self.ident = torch.where(mask[..., None], e, self.ident)
        n_new = int(mask.sum().item())
        ids = torch.zeros_like(self.gid)
        ids[mask] = torch.arange(self.next_identity, self.next_identity + n_new, device=self.device)
        self.gid = torch.where(mask, ids, self.gid)
        self.next_identity += n_new

    def _advance(self):
        if self.frame > 0:
            self.cx = self.cx + self.vx
            self.cy = self.cy + self.vy
            out = (self.cx < 0) | (self.cx >= IMAGE_W) | (self.cy < 0) | (self.cy >= IMAGE_H)
            if bool(out.any()):
                self._respawn(out)
        if self.truth is not None:
            w = self.h * self.cfg.aspect
            box = torch.stack([self.cx - w / 2.0, self.cy - self.h / 2.0, w, self.h], dim=-1)
            self.truth.append((self.frame, self.active.clone(), self.gid.clone(), box))
        self.frame += 1

    def record_truth(self) -> None:
        """Keep the ground truth of every frame generated from now on: all
        active objects (occlusion dropouts included -- the detector misses them,
        the scene still holds them), image-space tlwh, identity ids."""
        self.truth = []

    def truth_frames(self, stream: int = 0) -> dict:
        """Ground truth of one stream as moteval frame boxes {frame: [(id, BoundingBox)]}."""
        from .core import BoundingBox
        out = {}
        for frame, active, gid, box in self.truth or []:
            sel = active[stream]
            ids = gid[stream][sel].tolist()
            bx = box[stream][sel].tolist()
            out[frame] = [(int(i), BoundingBox(*b)) for i, b in zip(ids, bx)]
        return out

    def alloc(self, frames: int):
        """Empty head / embedding tensors for ``frames`` frames (embeddings channels_last)."""
        heads, embs = [], []
        for s in STRIDES:
            H, W = GRID[s]
            heads.append(torch.empty(frames, 24, H, W, dtype=torch.float32, device=self.device))
            embs.append(torch.empty(frames, self.cfg.dim, H, W, dtype=torch.float32, device=self.device,
                                    memory_format=torch.channels_last))
        return HeadOutputs(tuple(heads), tuple(embs))

    def _background(self, out: HeadOutputs):
        D = self.cfg.dim
        for head, emb in zip(out.heads, out.embs):
            head.normal_(0.0, 1.0, generator=self.gen)
            head[:, 4::6] = 0.0
            head[:, 5::6] -= 4.0
            emb.normal_(0.0, 1.0 / math.sqrt(D), generator=self.gen)

    def next_batch(self, B: int | None = None, out: HeadOutputs | None = None) -> HeadOutputs:
        """Advance all streams by B frames; frames are stream-major (f = s*B + b)."""
        c = self.cfg
        B = c.batch if B is None else B
        S, N = self.active.shape
        F = S * B
        out = out or self.alloc(F)
        self._background(out)
        for b in range(B):
            self._advance()
            vis = self.active & (self._rand(S, N) >= c.p_miss)
            self._encode(out, vis, b, B)
        return out

    def _encode(self, out: HeadOutputs, vis, b: int, B: int):
        c = self.cfg
        S, N = vis.shape
        s_idx, o_idx = torch.nonzero(vis, as_tuple=True)           # ascending object order per stream
        if s_idx.numel() == 0:
            return
        frame = s_idx * B + b
        cx = self.cx[s_idx, o_idx] * self.r + self.pad_x
        cy = self.cy[s_idx, o_idx] * self.r + self.pad_y
        h = self.h[s_idx, o_idx] * self.r
        w = self.h[s_idx, o_idx] * c.aspect * self.r
        inter = torch.minimum(w[:, None], self.an_w[None]) * torch.minimum(h[:, None], self.an_h[None])
        iou = inter / (w[:, None] * h[:, None] + self.an_w[None] * self.an_h[None] - inter)
        best = torch.argmax(iou, dim=1)
        si, a = self.an_si[best], self.an_a[best]
        aw, ah = self.an_w[best], self.an_h[best]
        n = cx.numel()
        noise = c.delta_sigma * self._randn(n, 4)
        if c.literal_noise:
            en = c.emb_sigma * self._randn(n, c.dim, dtype=torch.float32)
        else:
            en = (c.emb_sigma / math.sqrt(c.dim)) * self._randn(n, c.dim, dtype=torch.float32)
        emb_val = self.ident[s_idx, o_idx] + en
        seq = torch.arange(n, device=self.device)
        for k, stride in enumerate(STRIDES):
            sel = si == k
            if not bool(sel.any()):
                continue
            H, W = GRID[stride]
            gx = torch.clamp(torch.floor(cx[sel] / stride), 0, W - 1)
            gy = torch.clamp(torch.floor(cy[sel] / stride), 0, H - 1)
            fx = torch.clamp(cx[sel] / stride - gx, 1e-3, 1 - 1e-3)
            fy = torch.clamp(cy[sel] / stride - gy, 1e-3, 1 - 1e-3)
            t = torch.stack([torch.log(fx / (1 - fx)), torch.log(fy / (1 - fy)),
                             torch.log(w[sel] / aw[sel]), torch.log(h[sel] / ah[sel])], dim=1) + noise[sel]
            fr, aa, gxi, gyi, q = frame[sel], a[sel], gx.long(), gy.long(), seq[sel]
            # collision rule: the later object (higher sequence number) wins, deterministically
            akey = ((fr * 4 + aa) * H + gyi) * W + gxi
            win = torch.full((int(akey.max().item()) + 1,), -1, dtype=torch.long, device=self.device)
            win.scatter_reduce_(0, akey, q, reduce="amax")
            keep = win[akey] == q
            head = out.heads[k]
            for ch in range(4):
                head[fr[keep], 6 * aa[keep] + ch, gyi[keep], gxi[keep]] = t[keep, ch].float()
            head[fr[keep], 6 * aa[keep] + 4, gyi[keep], gxi[keep]] = -4.0
            head[fr[keep], 6 * aa[keep] + 5, gyi[keep], gxi[keep]] = 4.0
            ckey = (fr * H + gyi) * W + gxi
            cwin = torch.full((int(ckey.max().item()) + 1,), -1, dtype=torch.long, device=self.device)
            cwin.scatter_reduce_(0, ckey, q, reduce="amax")
            ck = cwin[ckey] == q
            emb = out.embs[k]
            # [F, D, H, W] channels_last: assign per detection row over D
            emb.permute(0, 2, 3, 1)[fr[ck], gyi[ck], gxi[ck]] = emb_val[q[ck]]


def make(name: str, device="cuda", **overrides) -> HeadSynth:
    return HeadSynth(replace(CONFIGS[name], **overrides), device)
