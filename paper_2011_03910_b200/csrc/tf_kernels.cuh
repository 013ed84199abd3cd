// Device-buffer descriptors and host launchers shared by tf_kernels.cu and tf_capi.cu.
#pragma once

#include "tf_device.cuh"

namespace tfd {

constexpr int kAssocThreads = 256;
constexpr int kAssocThreadsSmall = 128;   // two association CTAs per SM (many streams)
constexpr int kFidxInline = 32;           // frame indices passed in the launch parameters

// Per-frame detection buffer written by the frame stage, read by associate_kernel.
// Arrays are [frames][cap_det] (meas: x4, emb: xD).
struct DetBuf {
  int* count;        // [F] kept detections
  int* cand_count;   // [F] candidates past the confidence test
  int* status;       // [F] tf_status of the frame stage
  double* meas;      // (cx, cy, a, h) of each kept detection
  double* obj;       // objectness
  int* code;         // global anchor index (heads) / input row (dets)
  float* emb;        // unit embedding (fp32)
};

// Per-stream track tables, [streams][cap_tracks] in list order (= id order).
struct TrackBuf {
  long long* id;
  int* state;        // 0 ACTIVE, 1 LOST
  int* hits;
  long long* lost;   // -1 = None
  long long* last;
  int* slot;         // embedding slot in emb_pool
  double* mean;      // [8]
  double* cov;       // [12]: per axis (pp, pv, vv)
  float* emb_pool;   // [streams][cap_tracks][D]
  int* free_stack;   // [streams][cap_tracks]
  int* n_free;       // [streams]
  int* n_tracks;     // [streams]
  long long* next_id;
  long long* last_frame;
  int* status;       // [streams]: (frame << 8) | tf_status of the last update, 0 ok
};

struct OutBuf {
  int* count;
  long long* track_id;
  double* box;
  double* objectness;
  int max_records;
};

struct TraceBuf {
  int* cand_count;
  int* det_count;
  int* det_code;
  long long* det_track;
  double* det_cost;
  int* det_matched;
};

constexpr int kPhaseSlots = 40;   // associate_kernel phase timers / counters (tf_phase_stats)

struct AssocArgs {
  DetBuf det;
  TrackBuf trk;
  OutBuf out;
  TraceBuf trace;
  const long long* frame_index;  // [F] device (frames >= n_fidx_inline)
  int n_fidx_inline;             // small updates pass their frame indices by value ...
  long long fidx_inline[kFidxInline];   // ... (no per-update host->device copy)
  int stream_begin, B;
  int cap_tracks, cap_det, cap_entries;
  int16_t* pool_col;             // [streams][cap_tracks * cap_det] overflow CSR
  int16_t* pool_row;
  double* pool_val;
  int16_t* pool_aux;             // [streams][2 * cap_tracks * cap_det] overflow edge lists
  long long* stats;              // [kPhaseSlots] phase cycles / counters (nullptr = off)
  const int* order_in;           // [n_streams] block -> local stream (longest first), nullptr = identity
  int* order_out;                // written by the last CTA for the next launch over these streams (C == 1)
  long long* work;               // [n_streams] per-stream frame-loop cycles of this launch (order_out)
  unsigned* ticket;              // CTA completion counter (order_out), left at 0
  const unsigned* ready;         // overlapped mode: [F] frame f decoded when ready[f] == epoch (nullptr: off)
  unsigned epoch;
  long long* sclk;               // [streams][4] leader globaltimer: entry, prologue done, frames done, exit (nullptr = off)
  int cluster;                   // CTAs per stream (1 = no cluster)
  int threads;                   // kAssocThreads, or kAssocThreadsSmall (no cluster)
  int zero_smem;                 // diagnostics (TF_ZERO_SMEM): clear the dynamic shared memory at launch
};

struct HeadLaunch {
  const tf_heads* heads;
  const float* head_ptr[3];      // device-visible head tensors (staged copy for host input)
  const float* emb_ptr[3];       // device-visible embedding maps (mapped host memory for host input)
  const float* delta_ptr[3];     // device-visible box deltas (same tensor as head_ptr for device input)
  long long delta_stride_n[3], delta_stride_c[3];
  int frames, cap_cand, cap_det;
  DetBuf det;
  // overlapped decode + association (frame_heads_kernel overlapped mode); ready == nullptr: off
  unsigned* ready;
  unsigned epoch;
  int* ticket;
  const int* order;
  int first_wave, streams, B, persist_ctas;
};

size_t frame_smem_bytes(int total_anchors, int cap_cand);
// static shared memory of associate_kernel (budgeted next to the dynamic plan)
size_t assoc_static_smem();
size_t assoc_smem_bytes(int cap_tracks, int cap_det, int cap_entries);

cudaError_t launch_frame_heads(const HeadLaunch& h, const Params& P, cudaStream_t st);
cudaError_t launch_frame_dets(const double* boxes, const double* obj, const float* emb, const uint8_t* has, int n,
                              int cap_cand, int cap_det, const DetBuf& det, const Params& P, cudaStream_t st);
// Batched already-decoded rows (detection-file source): one CTA per frame,
// rows of frame f at [offsets[f], offsets[f+1]), parse_output normalisation.
cudaError_t launch_frame_rows(const double* boxes, const double* obj, const float* emb, const int* offsets,
                              int frames, int normalize, int cap_cand, int cap_det, const DetBuf& det,
                              const Params& P, cudaStream_t st);
cudaError_t launch_associate(const AssocArgs& a, int n_streams, const Params& P, cudaStream_t st);
int assoc_cluster_size(int n_streams, int cap_tracks, int cap_det, int cap_entries);
cudaError_t launch_nms_sets(int n_sets, const int* offsets, const double* boxes, const double* scores,
                            const double* thr, uint8_t* keep, int* status, int cap, cudaStream_t st);
cudaError_t launch_lap_dense(int n, const int* shapes, const long long* cost_off, const double* costs,
                             const long long* row_off, int* col_for_row, int* status, int cap_n,
                             int16_t* pool_col, double* pool_val, int* pool_rowptr, long long pool_stride,
                             cudaStream_t st);
cudaError_t launch_kalman(int op, int n, const Params& P, const double* mi, const double* ci, const double* z,
                          double* mo, double* co, int* status, cudaStream_t st);
cudaError_t launch_gating(int nt, const double* means, const double* covs, int nm, const double* z, int metric,
                          const Params& P, double* out, int* status, cudaStream_t st);
cudaError_t launch_cosine_cost(int nt, int nd, int dim, const float* te, const float* de, double* out,
                               cudaStream_t st);
cudaError_t launch_normalize_rows(int n, int dim, const double* in64, const float* in32, long long stride,
                                  int quantize, float* out, int* status, cudaStream_t st);
cudaError_t launch_binary16(long long n, const float* in, float* out, int* status, cudaStream_t st);
cudaError_t launch_smooth(int n, int dim, const float* o, const float* q, double alpha, double beta, float* out,
                          int* status, cudaStream_t st);
cudaError_t launch_iou(int n, const double* a, const double* b, double* out, cudaStream_t st);

// MOT evaluation (tf_moteval.cu)
size_t mot_accumulate_smem(int cap_g, int cap_h, int cap_e);
cudaError_t launch_mot_accumulate(int frames, const int* gt_ptr, const int* gt_id, const double* gt_box,
                                  const int* hyp_ptr, const int* hyp_id, const double* hyp_box, int n_gt_ids,
                                  int n_hyp_ids, double iou_min, int cap_g, int cap_h, int cap_e, int* prev, int* hpos,
                                  int* match_count, int* match_gt, int* match_hyp, double* match_iou,
                                  uint8_t* gt_matched, uint8_t* hyp_matched, int* status, cudaStream_t st);
cudaError_t launch_mot_coverage(int frames, const int* gt_ptr, const int* gt_id, const double* gt_box,
                                const int* hyp_ptr, const int* hyp_id, const double* hyp_box, double iou_min,
                                int n_hyp_ids, int* coverage, cudaStream_t st);

}  // namespace tfd
