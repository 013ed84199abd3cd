"""Constant-velocity Kalman filter (mirror of tf/motion.py) on the GPU.

``KalmanFilter`` keeps the reference's value-in/value-out API on
``KalmanState`` (mean[8], covariance[8x8]); each call launches the dense 8x8
kernel (tf_kalman / tf_gating). The ``*_batch`` methods run any number of
states in one launch. The tracking path uses the compact exact form of the
same filter inside associate_kernel (tf_device.cuh, struct KF).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import InvalidMeasurementError, NumericError

CHI2_GATE_95_4DOF = 9.4877   # tf/motion.py:23

_OP = {"initiate": 0, "predict": 1, "project": 2, "update": 3}


@dataclass(frozen=True)
class MotionNoise:
    """Noise weights (tf/motion.py:28-41)."""

    std_weight_position: float = 1.0 / 20
    std_weight_velocity: float = 1.0 / 160
    std_aspect: float = 1e-2
    std_aspect_velocity: float = 1e-5
    std_aspect_measurement: float = 1e-1


@dataclass(frozen=True)
class KalmanState:
    """Gaussian state (tf/motion.py:44-49)."""

    mean: np.ndarray
    covariance: np.ndarray


def _config(noise: MotionNoise) -> _lib.TfConfig:
    return _lib.TfConfig(0.5, 0.4, 0.7, CHI2_GATE_95_4DOF, 0.9, noise.std_weight_position,
                         noise.std_weight_velocity, noise.std_aspect, noise.std_aspect_velocity,
                         noise.std_aspect_measurement, 0, 30, 1, 512, 0, 0)


class KalmanFilter:
    """Predict / update cycle (tf/motion.py:52-142), executed on the GPU."""

    def __init__(self, noise: MotionNoise | None = None) -> None:
        self.noise = noise or MotionNoise()
        self._cfg = _config(self.noise)

    # -- batched device entry points -----------------------------------------
    def _run(self, op: str, means, covs, zs):
        torch = _lib.require_cuda()
        lib = _lib.load()
        n = (zs if zs is not None else means).shape[0]
        dm = None if means is None else torch.as_tensor(np.ascontiguousarray(means, np.float64)).cuda()
        dc = None if covs is None else torch.as_tensor(np.ascontiguousarray(covs, np.float64)).cuda()
        dz = None if zs is None else torch.as_tensor(np.ascontiguousarray(zs, np.float64)).cuda()
        proj = op == "project"
        mo = torch.empty(n, 4 if proj else 8, dtype=torch.float64, device="cuda")
        co = torch.empty(n, *(4, 4) if proj else (8, 8), dtype=torch.float64, device="cuda")
        st = torch.zeros(n, dtype=torch.int32, device="cuda")
        _lib.check(lib.tf_kalman(_OP[op], n, self._cfg, _lib.ptr(dm), _lib.ptr(dc), _lib.ptr(dz),
                                 mo.data_ptr(), co.data_ptr(), st.data_ptr(), _lib.stream_handle()))
        status = st.cpu().numpy()
        if status.any():
            code = int(status[status != 0][0])
            if code == 2:
                raise InvalidMeasurementError("measurement height must be positive")
            raise NumericError("innovation covariance is singular") if code == 9 else _lib.status_error(code, op)
        return mo.cpu().numpy(), co.cpu().numpy()

    def initiate_batch(self, zs: np.ndarray):
        return self._run("initiate", None, None, np.atleast_2d(zs))

    def predict_batch(self, means: np.ndarray, covs: np.ndarray):
        return self._run("predict", means, covs, None)

    def project_batch(self, means: np.ndarray, covs: np.ndarray):
        return self._run("project", means, covs, None)

    def update_batch(self, means: np.ndarray, covs: np.ndarray, zs: np.ndarray):
        return self._run("update", means, covs, zs)

    # -- reference API -------------------------------------------------------
    def initiate(self, measurement: np.ndarray) -> KalmanState:
        z = np.asarray(measurement, dtype=np.float64).reshape(1, 4)
        if float(z[0, 3]) <= 0:
            raise InvalidMeasurementError(f"measurement height must be positive, got {float(z[0, 3])}")
        m, c = self.initiate_batch(z)
        return KalmanState(mean=m[0], covariance=c[0])

    def predict(self, state: KalmanState) -> KalmanState:
        m, c = self.predict_batch(state.mean[None], state.covariance[None])
        return KalmanState(mean=m[0], covariance=c[0])

    def project(self, state: KalmanState) -> tuple[np.ndarray, np.ndarray]:
        m, c = self.project_batch(state.mean[None], state.covariance[None])
        return m[0], c[0]

    def update(self, state: KalmanState, measurement: np.ndarray) -> KalmanState:
        m, c = self.update_batch(state.mean[None], state.covariance[None],
                                 np.asarray(measurement, np.float64)[None])
        return KalmanState(mean=m[0], covariance=c[0])

    def gating_distance(self, state: KalmanState, measurements: np.ndarray) -> np.ndarray:
        """Squared Mahalanobis distance to each of N measurements (tf/motion.py:128-142)."""
        return gate_matrix(np.asarray(state.mean)[None], np.asarray(state.covariance)[None],
                           np.atleast_2d(np.asarray(measurements, np.float64)), "mahalanobis", self.noise)[0]


def gate_matrix(means: np.ndarray, covs: np.ndarray, measurements: np.ndarray, metric: str,
                noise: MotionNoise | None = None) -> np.ndarray:
    """[T, N] gate values (Tracker._gate_matrix, tf/tracker.py:161-170) in one launch."""
    from .errors import ConfigError

    torch = _lib.require_cuda()
    metric_code = {"mahalanobis": 0, "euclidean": 1}.get(metric)
    if metric_code is None:
        raise ConfigError(f"unknown gate metric {metric!r}")
    nt, nm = means.shape[0], measurements.shape[0]
    out = torch.empty(nt, nm, dtype=torch.float64, device="cuda")
    if nt == 0 or nm == 0:
        return out.cpu().numpy()
    dm = torch.as_tensor(np.ascontiguousarray(means, np.float64)).cuda()
    dc = torch.as_tensor(np.ascontiguousarray(covs, np.float64)).cuda()
    dz = torch.as_tensor(np.ascontiguousarray(measurements, np.float64)).cuda()
    st = torch.zeros(nt, dtype=torch.int32, device="cuda")
    _lib.check(_lib.load().tf_gating(nt, dm.data_ptr(), dc.data_ptr(), nm, dz.data_ptr(), metric_code,
                                     _config(noise or MotionNoise()), out.data_ptr(), st.data_ptr(),
                                     _lib.stream_handle()))
    if int(st.max().item()) != 0:
        raise NumericError("projected covariance is singular")
    return out.cpu().numpy()
