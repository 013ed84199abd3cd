/*
 * trackforge_b200 - C ABI of the B200-native decode -> NMS -> association path.
 *
 * Drop-in boundary for the reference's per-frame post-processing
 * (trackforge 0.1.0, /root/reference/pkg/src/trackforge; "tf/" below). The
 * reference is pure Python and has no FFI of its own; these entry points are
 * what its ctypes binding would call (INTEGRATION.md shows that stub). Every
 * signature uses plain pointers and sizes; no torch types cross the boundary.
 *
 * Conventions
 *  - Pointers are device pointers unless a field says "host". Calls are
 *    asynchronous on the caller's CUDA stream (`stream`, a cudaStream_t) unless
 *    documented as synchronising.
 *  - Every function returns a tf_status. TF_OK == 0. Codes 1..9 map one to one
 *    onto the reference exception classes of tf/errors.py (names in
 *    tf_status_name()); 10.. are boundary-only conditions.
 *  - Inputs are borrowed for the duration of the call (until the work queued on
 *    `stream` completes); outputs go to caller-allocated buffers.
 *  - A context serves one device; calls on one context must be serialised by
 *    the caller, mirroring the reference's single-owner Tracker contract
 *    (SPEC.md:415).
 */
#ifndef TRACKFORGE_B200_H
#define TRACKFORGE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes. 1..9 <-> tf/errors.py classes. */
typedef enum tf_status {
  TF_OK = 0,
  TF_INVALID_BOX = 1,            /* InvalidBoxError            tf/errors.py:12 */
  TF_INVALID_MEASUREMENT = 2,    /* InvalidMeasurementError    tf/errors.py:16 */
  TF_DIMENSION = 3,              /* DimensionError             tf/errors.py:20 */
  TF_DEGENERATE_EMBEDDING = 4,   /* DegenerateEmbeddingError   tf/errors.py:24 */
  TF_PRECISION_OVERFLOW = 5,     /* PrecisionOverflowError     tf/errors.py:28 */
  TF_LAYOUT = 6,                 /* LayoutError                tf/errors.py:32 */
  TF_CONFIG = 7,                 /* ConfigError                tf/errors.py:48 */
  TF_ORDERING = 8,               /* OrderingError              tf/errors.py:52 */
  TF_NUMERIC = 9,                /* NumericError               tf/errors.py:56 */
  TF_CAPACITY = 10,              /* a fixed device capacity was exceeded (never a silent drop) */
  TF_CUDA = 11,                  /* CUDA runtime failure */
  TF_ARGUMENT = 12               /* invalid argument at the boundary */
} tf_status;

/* TrackerConfig (tf/tracker.py:43-56) + MotionNoise (tf/motion.py:28-41)
 * + the MIXED-precision switch of the pipeline (tf/pipeline.py:436-441). */
typedef struct tf_config {
  double conf_threshold;          /* filter_confidence, tf/postproc.py:61-65 */
  double nms_iou;                 /* nms, tf/postproc.py:68-89 */
  double max_cost;                /* match_with_threshold, tf/assoc.py:90-107 */
  double gate_threshold;          /* apply_gate, tf/assoc.py:49-57 (default 9.4877) */
  double smoothing_alpha;         /* smooth_embedding, tf/tracker.py:67-71 */
  double std_weight_position;     /* 1/20 */
  double std_weight_velocity;     /* 1/160 */
  double std_aspect;              /* 1e-2 */
  double std_aspect_velocity;     /* 1e-5 */
  double std_aspect_measurement;  /* 1e-1 */
  int32_t gate_metric;            /* 0 = "mahalanobis", 1 = "euclidean" (tf/tracker.py:161-170) */
  int32_t max_lost;               /* 30 */
  int32_t min_hits;               /* 1 */
  int32_t embedding_dim;          /* 512; any D >= 1 */
  int32_t quantize_binary16;      /* 1 = MIXED: fp16-quantise + renormalise detection embeddings */
  /* JDE extensions the reference does not have (SURVEY.md section 8 name
   * map; off = the reference path, parity with the reference). Zero-filled
   * fields keep them off. */
  int32_t iou_stage;              /* 1: second association stage on 1 - IoU for tracks ACTIVE before the
                                     frame and detections left unmatched, pairs above iou_threshold dissolved */
  double motion_lambda;           /* lambda-fused cost lambda * cosine + motion_weight * gate distance ... */
  double motion_weight;           /* ... with motion_weight = 1 - lambda (as the caller computes it); 0 = off */
  double iou_threshold;           /* second-stage threshold on 1 - IoU (JDE: 0.5) */
} tf_config;

/* Fixed device capacities. Exceeding one returns TF_CAPACITY. */
typedef struct tf_capacity {
  int32_t streams;                /* independent tracker instances in this context */
  int32_t max_frames;             /* max frames per update call (streams x B) */
  int32_t max_candidates;         /* per frame, after the confidence test (<= 1024) */
  int32_t max_detections;         /* per frame, after NMS (<= 1024) */
  int32_t max_tracks;             /* per stream, ACTIVE + LOST (<= 1024) */
  int32_t reserved;
} tf_capacity;

/* One YOLO head scale (JDE layout). `head` is [N, 24, H, W] fp32 with channel
 * 6a+k for anchor a: k = 0..3 box deltas, 4 background logit, 5 foreground
 * logit; each channel plane must be H*W contiguous (h stride W, w stride 1).
 * `emb` is [N, D, H, W] fp32 with arbitrary element strides (channels_last,
 * i.e. stride_c == 1, is the fast path). Anchors are (w, h) pairs in input
 * pixels. `stride` is the scale's pixel stride (32, 16 or 8). `channels` is
 * the embedding map's channel count D; tf_update_heads returns TF_LAYOUT
 * unless it equals tf_config.embedding_dim (parse_output's row-width check,
 * tf/postproc.py:25-29). */
typedef struct tf_head_scale {
  const float* head;
  int64_t head_stride_n, head_stride_c;
  const float* emb;
  int64_t emb_stride_n, emb_stride_c, emb_stride_h, emb_stride_w;
  int32_t height, width, stride, channels;
  float anchors[8];
} tf_head_scale;

/* Three scales in candidate order (stride 32, 16, 8), plus the letterbox that
 * maps 1088x608 input pixels back to image pixels: image = (v - pad) * scale_inv. */
typedef struct tf_heads {
  tf_head_scale scale[3];
  double scale_inv, pad_x, pad_y;
  int32_t host_memory;            /* 1: head/emb are pinned HOST pointers (read zero-copy) */
  int32_t dtype;                  /* element type of head and emb: 0 fp32, 1 binary16 (MIXED
                                     input mode; the pointers then address __half data and the
                                     strides count __half elements) */
} tf_heads;

/* Per-frame records = TrackerOutput.records (tf/tracker.py:59-64,159):
 * (track_id, tlwh box, objectness), sorted by id. Frame f of an update is
 * stream-major: f = local_stream * B + b. All arrays are [frames][max_records]
 * (box: [frames][max_records][4]). With tf_heads.host_memory the record
 * buffers are host pointers too. */
typedef struct tf_records {
  int32_t* count;
  int64_t* track_id;
  double* box;
  double* objectness;
  int32_t max_records;
  int32_t reserved;
} tf_records;

/* Optional per-frame parity trace (any pointer may be NULL), [frames][max_detections]:
 *  cand_count[f]      candidates that passed the confidence test (decode output)
 *  det_count[f]       detections kept by NMS
 *  det_code[f][k]     kept detection k: global anchor index (heads) or input row (dets)
 *  det_track[f][k]    track id detection k was matched to or born as
 *  det_cost[f][k]     gated cosine cost of the match (NaN for births)
 *  det_matched[f][k]  1 matched, 0 born                                        */
typedef struct tf_trace {
  int32_t* cand_count;
  int32_t* det_count;
  int32_t* det_code;
  int64_t* det_track;
  double* det_cost;
  int32_t* det_matched;
} tf_trace;

/* Host-side export of one stream's track table (Tracker.tracks, tf/tracker.py:79;
 * Track fields tf/tracker.py:30-40). Arrays hold max_tracks entries; covariance is
 * expanded to 8x8. lost_since == -1 encodes None. */
typedef struct tf_track_export {
  int32_t count;
  int32_t reserved;
  int64_t next_id;                /* ids 1..next_id-1 issued; removed = issued - live */
  int64_t last_frame;             /* INT64_MIN when no frame was stepped */
  int64_t* track_id;
  int32_t* state;                 /* 0 ACTIVE, 1 LOST */
  int32_t* hits;
  int64_t* lost_since;
  int64_t* last_update_frame;
  double* mean;                   /* [count][8] */
  double* covariance;             /* [count][8][8] */
  float* embedding;               /* [count][D] */
} tf_track_export;

typedef struct tf_ctx tf_ctx;

/* ---- context ---------------------------------------------------------- */
int tf_version(void);
const char* tf_status_name(int status);
int tf_create(const tf_config* config, const tf_capacity* capacity, int32_t device, tf_ctx** out);
int tf_destroy(tf_ctx* ctx);
const char* tf_last_error(const tf_ctx* ctx);
int tf_reset_stream(tf_ctx* ctx, int32_t stream, void* cuda_stream);

/* Batched update(head_outputs) -> online_tracks for streams
 * [stream_begin, stream_begin + n_streams), B frames each. `frame_index` is a
 * HOST array [n_streams * B]; each stream's indices must strictly increase
 * past its last stepped frame (OrderingError, tf/tracker.py:87-91). Replaces
 * parse_output + Tracker.step per frame (tf/pipeline.py:291-302). Errors found
 * on the device are reported by tf_finish(). */
int tf_update_heads(tf_ctx* ctx, const tf_heads* heads, int32_t stream_begin, int32_t n_streams,
                    int32_t frames_per_stream, const int64_t* frame_index,
                    const tf_records* out, const tf_trace* trace, void* cuda_stream);

/* Tracker.step(frame_index, detections) for one stream (tf/tracker.py:85-159)
 * on already-parsed detections: boxes [n][4] tlwh fp64, objectness [n] fp64,
 * embeddings [n][D] fp32 (used as given, like Detection.embedding),
 * has_embedding [n] (0 -> DimensionError if the detection survives NMS).
 * Device pointers. */
/* Batched post-decode entry (the detection-file source, tf/detgen.py:366-484,
 * fed through parse_output + Tracker.step, tf/pipeline.py:291-302): S streams x
 * B frames (stream-major) of already-decoded rows. Frame f's rows are
 * [row_offsets[f], row_offsets[f+1]) (HOST array of F + 1) of the DEVICE arrays
 * boxes [N][4] tlwh, objectness [N] and embeddings [N][D] fp32. With
 * normalized = 0 the embeddings are raw row values and are normalised here as
 * parse_output does (DegenerateEmbeddingError on any row); with 1 they are
 * parse_output's unit vectors already (e.g. rows whose raw values are not fp32,
 * normalised by tf_normalize_rows from fp64). Records are written like
 * tf_update_heads'. Asynchronous on `cuda_stream`. */
int tf_update_detections(tf_ctx* ctx, int32_t stream_begin, int32_t n_streams, int32_t B,
                         const int64_t* frame_index, const int32_t* row_offsets, const double* boxes,
                         const double* objectness, const float* embeddings, int32_t normalized,
                         const tf_records* out, const tf_trace* trace, void* cuda_stream);

int tf_step_detections(tf_ctx* ctx, int32_t stream, int64_t frame_index, int32_t n,
                       const double* boxes, const double* objectness, const float* embeddings,
                       const uint8_t* has_embedding, const tf_records* out, const tf_trace* trace,
                       void* cuda_stream);

/* Synchronise `cuda_stream` (and the pipeline's side stream) and collect the
 * device-side errors of all update/step calls since the previous tf_finish.
 * Returns the first error (in stream, then frame order). */
int tf_finish(tf_ctx* ctx, void* cuda_stream);

/* Pipelining (the paper's PP stage overlap). When enabled,
 * tf_update_heads runs the decode of update i (H2D copies + frame kernel) on
 * the caller's stream and the association + outputs on a context-owned side
 * stream, with two detection-buffer sets, so the decode of update i+1 overlaps
 * the association of update i. Outputs of an update are valid after
 * tf_finish, or on any stream made to wait with tf_join. */
int tf_set_pipeline(tf_ctx* ctx, int32_t enabled);
int tf_join(tf_ctx* ctx, void* cuda_stream);

/* Copy one stream's tracks into caller HOST buffers (synchronising). */
int tf_export_tracks(tf_ctx* ctx, int32_t stream, tf_track_export* out, void* cuda_stream);

/* Inverse of tf_export_tracks (synchronising): make `in` (count tracks in
 * Tracker.tracks order, next_id, last_frame) stream's state, e.g. a reference
 * Tracker's tracks / _next_id / _last_frame at some frame (tf/tracker.py:74-83),
 * so a sequence resumes from it (parity bisection). TF_ARGUMENT for ids outside
 * [1, next_id) or repeated, a state other than 0/1, lost_since set for an
 * ACTIVE track (or -1 for a LOST one), or a covariance outside the per-axis
 * (position, velocity) form the filter keeps; TF_CAPACITY above max_tracks. */
int tf_import_tracks(tf_ctx* ctx, int32_t stream, const tf_track_export* in, void* cuda_stream);

/* Optional CUDA-event timing of the two kernels of every update (bench.py).
 * enabled: 0 off, 1 kernel events, 2 kernel events + the association
 * kernel's in-kernel phase timers (tf_phase_stats; they cost ~1% of the
 * kernel, so timed runs use 1); enabled | (N << 4) records the events on
 * every N-th update only (their host cost shows at small batches). tf_kernel_times synchronises, returns the
 * summed milliseconds of frame_heads_kernel and associate_kernel over the
 * updates since the last call, and resets the accumulators. */
int tf_set_profiling(tf_ctx* ctx, int32_t enabled);
int tf_kernel_times(tf_ctx* ctx, double* frame_ms, double* assoc_ms, int64_t* updates);
/* Number of kernels this context has launched since tf_create (update,
 * step and reset calls; bench.py reports the difference over its timed
 * region as gpu_launches). Host-side read, no synchronisation. */
int tf_launch_count(const tf_ctx* ctx, int64_t* launches);
/* Host->device copy milliseconds (pinned-host updates) summed over the window
 * read by the last tf_kernel_times call. */
int tf_copy_times(tf_ctx* ctx, double* h2d_ms);
/* Association launch shape (diagnostics): threads per CTA (256, or 128 with
 * two CTAs per SM for many streams) and CTAs per stream of the last update. */
int tf_launch_info(tf_ctx* ctx, int32_t* assoc_threads, int32_t* assoc_cluster);
/* Per-update event timeline since profiling was enabled (diagnostics): for
 * update u, out[6u..6u+5] = frame kernel start/end, association start/end,
 * host-input copy start/end in ms from the first update's copy start. */
int tf_timeline(tf_ctx* ctx, double* out, int32_t max_updates, int32_t* n_updates);
/* Per-phase SM cycles of associate_kernel summed over streams since profiling
 * was enabled (synchronising; resets): [0] load+predict [1] gate [2] CSR
 * [3] cosine cost [4] LAP [5] matches [6] Kalman update + EMA [7] records,
 * compaction, births; counters [8] tie fallbacks [9] finite entries
 * [10] multi-edge components [11] frames [12] sum T [13] sum K; LAP sub-phases
 * [16] components + tie check [17] peeling [18] residual components
 * [19] warp solves [20] full restatement (ties); why the full restatement
 * ran: [32] a component's uniqueness undecided (> 32 active rows) [33] an
 * alternative optimum [34] a star's runner-up within eps [35] entries beyond
 * the int16 edge lists. out has 40 entries. */
int tf_phase_stats(tf_ctx* ctx, int64_t* out40);
/* Per-stream association clocks of the last update run with profiling bit 2
 * (tf_set_profiling(ctx, 4 | ...); diagnostics, synchronising): out[4s..4s+3]
 * = the leader CTA's %globaltimer (ns) at entry, after the prologue (state
 * loaded), after the last frame, and at exit. n_streams <= the context's. */
int tf_stream_clocks(tf_ctx* ctx, int64_t* out, int32_t n_streams);
/* Benchmark support: hold `cuda_stream` until the host stores a non-zero
 * value into *flag (flag: host memory allocated mapped / pinned, passed as its
 * device alias), so that an update queued behind the hold runs with all of its
 * launches already queued (bench.py times single updates this way: the host's
 * submission time is reported beside the device time, not inside it). */
int tf_stream_hold(const volatile int32_t* flag, void* cuda_stream);

/* ---- stage-level entry points (batched; device pointers) ---------------- */

/* nms (tf/postproc.py:68-89) on n_sets independent sets. boxes [N][4] tlwh,
 * scores [N]; set i is rows [offsets[i], offsets[i+1]) with IoU threshold
 * thresholds[i]; keep [N] receives 1 for survivors. */
int tf_nms_sets(int32_t n_sets, const int32_t* offsets, const double* boxes, const double* scores,
                const double* thresholds, uint8_t* keep, int32_t* status, void* cuda_stream);

/* hungarian_solve (tf/assoc.py:60-87) on n matrices. Matrix i is rows x cols
 * = shapes[2i], shapes[2i+1], row-major fp64 at costs + cost_offsets[i]; +inf
 * marks forbidden edges. col_for_row receives, at row_offsets[i] + r, the
 * matched column of row r or -1. */
int tf_lap_dense(int32_t n, const int32_t* shapes, const int64_t* cost_offsets, const double* costs,
                 const int64_t* row_offsets, int32_t* col_for_row, int32_t* status, void* cuda_stream);

/* KalmanFilter (tf/motion.py:61-142) on n independent states, dense 8x8 form.
 * op: 0 initiate(z), 1 predict, 2 project (mean_out [n][4], cov_out [n][4][4]),
 * 3 update(z). */
int tf_kalman(int32_t op, int32_t n, const tf_config* config, const double* mean_in,
              const double* cov_in, const double* z, double* mean_out, double* cov_out,
              int32_t* status, void* cuda_stream);

/* gating_distance / Tracker._gate_matrix (tf/motion.py:128-142, tf/tracker.py:161-170):
 * out [n_tracks][n_meas]. metric 0 mahalanobis, 1 euclidean. */
int tf_gating(int32_t n_tracks, const double* means, const double* covs, int32_t n_meas,
              const double* z, int32_t metric, const tf_config* config, double* out,
              int32_t* status, void* cuda_stream);

/* build_cost_matrix (tf/assoc.py:34-46): out [nt][nd] = clip(1 - te.de^T, 0, 2) in fp64. */
int tf_cosine_cost(int32_t nt, int32_t nd, int32_t dim, const float* track_emb,
                   const float* det_emb, double* out, void* cuda_stream);

/* normalize (tf/core.py:100-111) of n rows of width dim; input fp64 (in64) or fp32
 * (in32, the other NULL). quantize != 0 applies quantize_binary16 + normalize again
 * (tf/pipeline.py:436-441). status[i] per row. */
int tf_normalize_rows(int32_t n, int32_t dim, const double* in64, const float* in32,
                      int64_t row_stride, int32_t quantize, float* out, int32_t* status,
                      void* cuda_stream);

/* quantize_binary16 (tf/core.py:124-136). status [n]. */
int tf_quantize_binary16(int64_t n, const float* in, float* out, int32_t* status, void* cuda_stream);

/* smooth_embedding (tf/tracker.py:67-71) of n row pairs. status [n]. */
int tf_smooth_embedding(int32_t n, int32_t dim, const float* old_emb, const float* new_emb,
                        double alpha, float* out, int32_t* status, void* cuda_stream);

/* iou (tf/core.py:71-80) of n box pairs. */
int tf_iou_pairs(int32_t n, const double* a, const double* b, double* out, void* cuda_stream);

/* ---- MOT evaluation of tracker outputs (tf/moteval.py) ----
 * All pointers DEVICE. Frames are the sorted union of gt and hypothesis frames;
 * rows of frame f are [gt_ptr[f], gt_ptr[f+1]) (resp. hyp_ptr), ids are dense
 * indices (< n_gt_ids / n_hyp_ids, unique within a frame), boxes tlwh fp64.
 *
 * tf_mot_accumulate = match_frame over every frame with the carried id mapping
 * (accumulate, tf/moteval.py:36-110): match i of frame f is stored at index
 * gt_ptr[f] + i (gt row, hyp row, IoU) in reference order (carried pairs in gt
 * order, then hungarian_solve pairs by row); gt_matched / hyp_matched flag the
 * rows. One CTA runs the frames in order; status[0] = TF_CAPACITY when a frame
 * exceeds max_gt / max_hyp / max_pairs (pairs with IoU >= iou_min). */
int tf_mot_accumulate(int32_t n_frames, const int32_t* gt_ptr, const int32_t* gt_id, const double* gt_box,
                      const int32_t* hyp_ptr, const int32_t* hyp_id, const double* hyp_box, int32_t n_gt_ids,
                      int32_t n_hyp_ids, int32_t max_gt_per_frame, int32_t max_hyp_per_frame,
                      int32_t max_pairs_per_frame, double iou_min, int32_t* match_count, int32_t* match_gt,
                      int32_t* match_hyp, double* match_iou, uint8_t* gt_matched, uint8_t* hyp_matched,
                      int32_t* status, void* cuda_stream);
/* Joint coverage of trajectory pairs for id_metrics (tf/moteval.py:196-232,
 * 337-345): coverage[gt id][hyp id] (zero-initialised by the caller, int32,
 * row-major n_gt_ids x n_hyp_ids) += frames where both are present with IoU >= iou_min. */
int tf_mot_coverage(int32_t n_frames, const int32_t* gt_ptr, const int32_t* gt_id, const double* gt_box,
                    const int32_t* hyp_ptr, const int32_t* hyp_id, const double* hyp_box, int32_t n_hyp_ids,
                    double iou_min, int32_t* coverage, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* TRACKFORGE_B200_H */
