"""Throughput of the stage kernels behind the reference's module API on large
batches (device-resident inputs, CUDA events): tf_kalman predict / update
(KalmanFilter batch API, dense 8x8 states), tf_normalize_rows, tf_iou_pairs.
Prints one JSON line per kernel with GB/s against MEASURED_PEAKS.json."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2011_03910_b200 import _lib  # noqa: E402
from paper_2011_03910_b200.motion import _OP, KalmanFilter  # noqa: E402

ROOT = Path(__file__).resolve().parents[1]
peak = 6545.0
try:
    mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    peak = float(mp.get("hbm_gbs", peak))
except Exception:
    pass
lib = _lib.load()
st = _lib.stream_handle()


def timed(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def report(name, n, nbytes, ms):
    gbs = nbytes / (ms / 1e3) / 1e9
    print(json.dumps({"kernel": name, "items": n, "ms": ms, "bytes": nbytes, "GBps": gbs, "peak_GBps": peak,
                      "frac": gbs / peak}), flush=True)


n = 1 << 20
kf = KalmanFilter()
g = torch.Generator(device="cuda").manual_seed(0)
means = torch.rand(n, 8, dtype=torch.float64, device="cuda", generator=g) * 100 + 50
covs = torch.zeros(n, 8, 8, dtype=torch.float64, device="cuda")
idx = torch.arange(8, device="cuda")
covs[:, idx, idx] = torch.rand(n, 8, dtype=torch.float64, device="cuda", generator=g) + 1.0
zs = means[:, :4] + 1.0
mo = torch.empty_like(means)
co = torch.empty_like(covs)
status = torch.zeros(n, dtype=torch.int32, device="cuda")
for op in ("predict", "update"):
    def run():
        _lib.check(lib.tf_kalman(_OP[op], n, kf._cfg, means.data_ptr(), covs.data_ptr(),
                                 zs.data_ptr() if op == "update" else None, mo.data_ptr(), co.data_ptr(),
                                 status.data_ptr(), st))
    ms = timed(run)
    nbytes = n * (72 * 8 * 2 + (32 if op == "update" else 0))
    report(f"kalman_kernel/{op}", n, nbytes, ms)

d = 512
rows = torch.randn(n // 4, d, dtype=torch.float32, device="cuda", generator=g)
out = torch.empty_like(rows)
st2 = torch.zeros(n // 4, dtype=torch.int32, device="cuda")
ms = timed(lambda: _lib.check(lib.tf_normalize_rows(n // 4, d, None, rows.data_ptr(), d, 0, out.data_ptr(),
                                                    st2.data_ptr(), st)))
report("normalize_rows_kernel", n // 4, (n // 4) * d * 8, ms)

a = torch.rand(n, 4, dtype=torch.float64, device="cuda", generator=g) * 100 + 1
b = a + 2.0
o = torch.empty(n, dtype=torch.float64, device="cuda")
ms = timed(lambda: _lib.check(lib.tf_iou_pairs(n, a.data_ptr(), b.data_ptr(), o.data_ptr(), st)))
report("iou_kernel", n, n * 72, ms)
