"""B200-native decode -> NMS -> association path of the JDE tracking pipeline.

Drop-in for trackforge's post-processing path (parse_output + Tracker.step,
/root/reference/pkg/src/trackforge): the same public names, argument meanings
and exception classes, with every compute step executed by hand-written
sm_100a CUDA kernels in libtrackforge_b200.so (C ABI: include/trackforge_b200.h).
There is no CPU fallback; compute entry points raise without the built
library or a CUDA device.
"""

from .errors import (  # noqa: F401
    CapacityError, ConfigError, ConsistencyError, CudaError, DegenerateEmbeddingError, DimensionError,
    DuplicateIdError, InvalidBoxError, InvalidMeasurementError, LayoutError, MeasurementError, NumericError,
    OrderingError, ParseError, PipelineAborted, PrecisionOverflowError, TrackforgeError, UndefinedMetricError,
)
from .core import (  # noqa: F401
    BINARY16_MAX, EMBEDDING_DIM, BoundingBox, Detection, box_to_measurement, cosine_distance, iou,
    measurement_to_box, normalize, quantize_binary16,
)
from .postproc import ROW_PREFIX, filter_confidence, nms, parse_output, serialize_detections  # noqa: F401
from .motion import CHI2_GATE_95_4DOF, KalmanFilter, KalmanState, MotionNoise  # noqa: F401
from .assoc import Assignment, apply_gate, build_cost_matrix, hungarian_solve, match_with_threshold  # noqa: F401
from .tracker import STrack, Track, Tracker, TrackerConfig, TrackerOutput, TrackState, smooth_embedding  # noqa: F401
from .engine import Capacity  # noqa: F401
from .heads import BatchTracker, HeadOutputs, OnlineTracks  # noqa: F401
from . import detfile  # noqa: F401  (detection-file source)
from . import moteval  # noqa: F401  (MOT rows and metrics of GPU outputs)

__version__ = "0.1.0"
