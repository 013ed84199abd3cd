// C ABI of trackforge_b200 (declared in include/trackforge_b200.h).
//
// Owns the device-resident per-stream track tables, the per-frame detection
// buffers and the launch sequence of one update:
//   [host input only] cudaMemcpy2DAsync of the 8 confidence planes per scale
//   frame_heads_kernel  (S*B CTAs)   decode + NMS + gather/normalise
//   associate_kernel    (S CTAs)     B frames per stream, sequential per stream
//   [host output only] cudaMemcpyAsync of the records
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "tf_kernels.cuh"

// NVTX ranges around the host entry points (SURVEY.md section 5 tracing: the
// reference's per-stage timers). A no-op unless a tool (ncu, nsys) injects.
namespace {
nvtxDomainHandle_t nvtx_domain() {
  static nvtxDomainHandle_t d = nvtxDomainCreateA("trackforge_b200");
  return d;
}
struct NvtxRange {
  explicit NvtxRange(const char* name) {
    nvtxEventAttributes_t a = {};
    a.version = NVTX_VERSION;
    a.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    a.messageType = NVTX_MESSAGE_TYPE_ASCII;
    a.message.ascii = name;
    nvtxDomainRangePushEx(nvtx_domain(), &a);
  }
  ~NvtxRange() { nvtxDomainRangePop(nvtx_domain()); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};
}  // namespace

using namespace tfd;

struct tf_ctx {
  tf_config cfg;
  tf_capacity cap;
  int device;
  Params P;
  std::string err;
  int cap_entries;
  int assoc_threads;              // 256, or 128 (two association CTAs per SM) for many streams
  // per-frame detection buffers
  DetBuf det;                 // = dets[0] (per-frame detection buffers)
  long long* d_frame_index;   // = d_fidx[0]
  int* d_row_offsets;         // [max_frames + 1] row ranges of tf_update_detections
  // pipelining (tf_set_pipeline): two buffer sets, decode on the caller's
  // stream, association + outputs on `side`
  DetBuf dets[2];
  long long* d_fidx[2];
  int pipeline, parity;
  cudaStream_t side;
  cudaEvent_t ev_dec[2], ev_asc[2];
  bool asc_pending[2];
  int touched_lo, touched_hi;
  // pinned staging ring for the per-update frame indices (a pageable H2D copy
  // may block the host and stall the pipeline)
  static constexpr int kRing = 4;
  long long* h_fidx[kRing];
  cudaEvent_t ev_fidx[kRing];
  bool fidx_used[kRing];
  int ring;
  // per-stream track tables
  TrackBuf trk;
  int16_t* pool_col;
  int16_t* pool_row;
  double* pool_val;
  int16_t* pool_aux;
  // host mirror of each stream's last stepped frame (ordering checks)
  std::vector<long long> last_frame;
  std::vector<long long> frame_scratch;
  // device staging used when inputs / outputs are host memory
  float* stage_conf[2][3];
  size_t stage_conf_elems[2][3];
  // device staging of host-output records, one set per pipeline parity; the
  // device->host copies run on their own stream so the next association
  // does not queue behind them
  int* rec_count[2];
  long long* rec_id[2];
  double* rec_box[2];
  double* rec_obj[2];
  cudaStream_t d2h;
  cudaEvent_t ev_d2h[2];
  bool d2h_pending[2];
  int rec_capacity;
  // streams touched by the last update (for tf_finish)
  int last_begin, last_count;
  // optional per-kernel CUDA-event timing (bench.py roofline)
  long long launches = 0;        // kernels launched by this context (tf_launch_count)
  int profiling;                 // bit 0 kernel events, bit 1 in-kernel phase timers
  int prof_stride = 1;            // events on every prof_stride-th update
  long long prof_counter = 0;
  bool prof_on = true;            // events for the current update
  std::vector<cudaEvent_t> events;   // triples: before frame kernel, after it, after associate
  size_t events_used;
  double last_h2d_ms;              // host->device copy time of the last tf_kernel_times window
  long long prof_bytes_frame, prof_frames;
  long long* d_stats;            // [kPhaseSlots] phase stats, then [streams][4] leader clocks (profiling bit 2)
  int n_streams_alloc = 0;
  int sms = 0;                    // SM count of the device
  // longest-first order of single-CTA streams over more than one wave (associate_kernel)
  int* d_order = nullptr;
  long long* d_work = nullptr;
  unsigned* d_ticket = nullptr;
  long long order_key = -1;       // (stream_begin, n_streams) the order in d_order was computed for
  int assoc_slots = 0;            // association CTAs resident at once
  bool env_no_lpt = false;        // TF_NO_LPT (read at tf_create): identity order
  // overlapped decode + association within one update (frame_heads_kernel overlapped mode)
  unsigned* d_ready = nullptr;    // [max_frames] per-frame decode flags (epoch values)
  int* d_fticket = nullptr;       // [2] the persistent decode grid's counters
  unsigned epoch = 0;
  bool env_overlap = false;       // TF_OVERLAP (read at tf_create): opt-in, see tf_update_heads
  int cluster_key, cluster_val;   // cached cluster size for the last stream count
  int env_cluster = 0;            // TF_CLUSTER (read at tf_create)
  bool env_zero_smem = false;     // TF_ZERO_SMEM (read at tf_create)
  std::vector<void*> allocs;
};

namespace {

const char* kNames[] = {"OK",
                        "InvalidBoxError",
                        "InvalidMeasurementError",
                        "DimensionError",
                        "DegenerateEmbeddingError",
                        "PrecisionOverflowError",
                        "LayoutError",
                        "ConfigError",
                        "OrderingError",
                        "NumericError",
                        "CapacityError",
                        "CudaError",
                        "ArgumentError"};

int fail(tf_ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  return code;
}

#define TF_CUDA(ctx, expr)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) return fail((ctx), TF_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
cudaError_t dev_alloc(tf_ctx* c, T** p, size_t n) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, n * sizeof(T) > 0 ? n * sizeof(T) : 16);
  if (e == cudaSuccess) {
    c->allocs.push_back(q);
    *p = static_cast<T*>(q);
  }
  return e;
}

Params make_params(const tf_config& c) {
  Params p;
  p.conf_threshold = c.conf_threshold;
  if (c.conf_threshold <= 0.0)
    p.conf_logit = -INFINITY;
  else if (c.conf_threshold >= 1.0)
    p.conf_logit = INFINITY;
  else
    p.conf_logit = std::log(c.conf_threshold) - std::log1p(-c.conf_threshold);
  p.nms_iou = c.nms_iou;
  p.max_cost = c.max_cost;
  p.gate_threshold = c.gate_threshold;
  p.alpha = c.smoothing_alpha;
  p.beta = 1.0 - c.smoothing_alpha;
  p.wp = c.std_weight_position;
  p.wv = c.std_weight_velocity;
  p.std_aspect = c.std_aspect;
  p.std_aspect_velocity = c.std_aspect_velocity;
  p.std_aspect_measurement = c.std_aspect_measurement;
  p.gate_metric = c.gate_metric;
  p.max_lost = c.max_lost;
  p.min_hits = c.min_hits;
  p.dim = c.embedding_dim;
  p.quantize = c.quantize_binary16;
  p.fuse = c.motion_weight != 0.0;
  p.lambda = c.motion_lambda;
  p.lambda_w = c.motion_weight;
  p.iou_stage = c.iou_stage != 0;
  p.iou_threshold = c.iou_threshold;
  return p;
}

// Configuration checks the reference performs on every step (filter_confidence
// tf/postproc.py:63-64, nms tf/postproc.py:76-77).
int check_step_config(tf_ctx* c) {
  const tf_config& g = c->cfg;
  if (!(g.conf_threshold >= 0.0 && g.conf_threshold <= 1.0))
    return fail(c, TF_CONFIG, "confidence threshold must be in [0, 1], got " + std::to_string(g.conf_threshold));
  if (!(g.nms_iou > 0.0 && g.nms_iou < 1.0))
    return fail(c, TF_CONFIG, "NMS IoU threshold must be in (0, 1), got " + std::to_string(g.nms_iou));
  if (g.motion_weight != 0.0 && !(g.motion_lambda >= 0.0 && g.motion_lambda <= 1.0))
    return fail(c, TF_CONFIG, "motion lambda must be in [0, 1], got " + std::to_string(g.motion_lambda));
  if (g.iou_stage && !(g.iou_threshold >= 0.0 && g.iou_threshold <= 1.0))
    return fail(c, TF_CONFIG, "second-stage IoU threshold must be in [0, 1], got " + std::to_string(g.iou_threshold));
  return TF_OK;
}

// benchmark support (tf_stream_hold): spin until the host releases the stream
// (gives up after 5 s, so a host that never releases cannot wedge the GPU)
__global__ void stream_hold_kernel(const volatile int32_t* flag) {
  if (threadIdx.x != 0) return;
  long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (*flag == 0) {
    __nanosleep(500);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 5000000000ll) break;
  }
}

__global__ void reset_streams_kernel(TrackBuf t, int s0, int n, int cap_tracks) {
  const int s = s0 + blockIdx.x;
  if (blockIdx.x >= n) return;
  for (int i = threadIdx.x; i < cap_tracks; i += blockDim.x)
    t.free_stack[static_cast<long long>(s) * cap_tracks + i] = cap_tracks - 1 - i;
  if (threadIdx.x == 0) {
    t.n_free[s] = cap_tracks;
    t.n_tracks[s] = 0;
    t.next_id[s] = 1;
    t.last_frame[s] = LLONG_MIN;
    t.status[s] = 0;
  }
}

int check_ordering(tf_ctx* c, int s, const long long* frames, int B) {
  long long prev = c->last_frame[s];
  for (int b = 0; b < B; ++b) {
    if (prev != std::numeric_limits<long long>::min() && frames[b] <= prev)
      return fail(c, TF_ORDERING, "stream " + std::to_string(s) + ": frame " + std::to_string(frames[b]) +
                                      " does not advance past " + std::to_string(prev));
    prev = frames[b];
  }
  return TF_OK;
}

TraceBuf to_trace(const tf_trace* t) {
  TraceBuf b{};
  if (t) {
    b.cand_count = t->cand_count;
    b.det_count = t->det_count;
    b.det_code = t->det_code;
    b.det_track = reinterpret_cast<long long*>(t->det_track);
    b.det_cost = t->det_cost;
    b.det_matched = t->det_matched;
  }
  // associate_kernel writes the per-detection trace only when all three exist
  if (!(b.det_track && b.det_cost && b.det_matched)) {
    b.det_track = nullptr;
    b.det_cost = nullptr;
    b.det_matched = nullptr;
  }
  return b;
}

__global__ void copy_codes_kernel(const int* count, const int* code, int* out, int frames, int cap_det) {
  const int f = blockIdx.x;
  if (f >= frames) return;
  const int n = count[f];
  for (int k = threadIdx.x; k < n; k += blockDim.x)
    out[static_cast<long long>(f) * cap_det + k] = code[static_cast<long long>(f) * cap_det + k];
}

// Stage host frame indices through the pinned ring and copy them to `dst`.
cudaError_t upload_frame_index(tf_ctx* c, long long* dst, const long long* src, int n, cudaStream_t st) {
  const int r = c->ring;
  c->ring = (c->ring + 1) % tf_ctx::kRing;
  cudaError_t e = cudaSuccess;
  if (c->fidx_used[r]) e = cudaEventSynchronize(c->ev_fidx[r]);
  if (e != cudaSuccess) return e;
  std::memcpy(c->h_fidx[r], src, sizeof(long long) * n);
  e = cudaMemcpyAsync(dst, c->h_fidx[r], sizeof(long long) * n, cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return e;
  c->fidx_used[r] = true;
  return cudaEventRecord(c->ev_fidx[r], st);
}

// cudaSetDevice only when another device is current (per-update host cost)
cudaError_t ensure_device(int device) {
  int cur = -1;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess || cur != device) e = cudaSetDevice(device);
  return e;
}

cudaError_t prof_mark(tf_ctx* c, int which, cudaStream_t st) {
  if (!c->profiling || !c->prof_on) return cudaSuccess;
  const size_t idx = c->events_used + which;
  while (c->events.size() <= idx) {
    cudaEvent_t e;
    cudaError_t r = cudaEventCreate(&e);   // timing events
    if (r != cudaSuccess) return r;
    c->events.push_back(e);
  }
  cudaError_t r = cudaEventRecord(c->events[idx], st);
  if (which == 3) c->events_used += 6;   // per update: frame, association, host->device copy
  return r;
}

}  // namespace

// Longest-first stream order for single-CTA association launches that need
// more than one wave of CTAs: the kernel's last CTA ranks the streams by their
// measured work for the next launch over the same streams (lpt_order).
static bool uses_stream_order(const tf_ctx* c, int cluster, int n_streams) {
  return cluster <= 1 && n_streams > c->assoc_slots && !c->env_no_lpt;
}
static long long order_key(int stream_begin, int n_streams) {
  return (static_cast<long long>(stream_begin) << 32) | static_cast<unsigned>(n_streams);
}
// the block order the next association over these streams will use (nullptr = identity)
static const int* next_stream_order(const tf_ctx* c, int cluster, int stream_begin, int n_streams) {
  return uses_stream_order(c, cluster, n_streams) && order_key(stream_begin, n_streams) == c->order_key ? c->d_order
                                                                                                        : nullptr;
}
static void set_stream_order(tf_ctx* c, AssocArgs& a, int stream_begin, int n_streams) {
  a.order_in = nullptr;
  a.order_out = nullptr;
  a.work = c->d_work;
  a.ticket = c->d_ticket;
  if (!uses_stream_order(c, a.cluster, n_streams)) {
    c->order_key = -1;
    return;
  }
  a.order_in = next_stream_order(c, a.cluster, stream_begin, n_streams);
  a.order_out = c->d_order;
  c->order_key = order_key(stream_begin, n_streams);
}

extern "C" {

int tf_version(void) { return 3; }   // 2: tf_head_scale.channels is checked; 3: tf_import_tracks

const char* tf_status_name(int status) {
  if (status < 0 || status > TF_ARGUMENT) return "UnknownError";
  return kNames[status];
}

const char* tf_last_error(const tf_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int tf_create(const tf_config* config, const tf_capacity* capacity, int32_t device, tf_ctx** out) {
  if (!config || !capacity || !out) return TF_ARGUMENT;
  *out = nullptr;
  const tf_capacity& k = *capacity;
  if (k.streams < 1 || k.max_frames < 1 || k.max_candidates < 1 || k.max_candidates > 1024 ||
      k.max_detections < 1 || k.max_detections > 1024 || k.max_tracks < 1 || k.max_tracks > 1024 ||
      config->embedding_dim < 1)
    return TF_ARGUMENT;
  tf_ctx* c = new tf_ctx();
  c->cfg = *config;
  c->cap = k;
  c->device = device;
  c->P = make_params(*config);
  c->last_begin = 0;
  c->last_count = 0;
  c->rec_capacity = 0;
  for (int b = 0; b < 2; ++b) {
    c->rec_count[b] = nullptr;
    c->d2h_pending[b] = false;
  }
  c->d2h = nullptr;
  c->profiling = 0;
  c->events_used = 0;
  c->prof_bytes_frame = 0;
  c->prof_frames = 0;
  c->cluster_key = -1;
  c->cluster_val = 1;
  {
    const char* ev = getenv("TF_CLUSTER");
    c->env_cluster = ev ? atoi(ev) & 63 : 0;
    c->env_zero_smem = getenv("TF_ZERO_SMEM") != nullptr;
  }
  for (int b = 0; b < 2; ++b)
    for (int i = 0; i < 3; ++i) {
      c->stage_conf[b][i] = nullptr;
      c->stage_conf_elems[b][i] = 0;
    }
  c->pipeline = 0;
  c->parity = 0;
  c->side = nullptr;
  c->asc_pending[0] = c->asc_pending[1] = false;
  c->touched_lo = 1 << 30;
  c->touched_hi = -1;
  c->ring = 0;
  for (int r = 0; r < tf_ctx::kRing; ++r) {
    c->h_fidx[r] = nullptr;
    c->fidx_used[r] = false;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    delete c;
    return TF_CUDA;
  }
  const size_t S = k.streams, F = k.max_frames, Km = k.max_detections, Tm = k.max_tracks,
               D = config->embedding_dim;
  // shared-memory budget for the association CTA decides how many CSR entries stay on chip
  int smem_optin = 0;
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  // keep as many gated entries on chip as the budget allows (the rest spill to a global pool)
  int entries = 8192;
  const size_t assoc_static = assoc_static_smem() + 256;
  int sms = 0, smem_sm = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  // Many streams (>= 2 per SM): two 128-thread association CTAs per SM when
  // the plan fits half of the SM's shared memory with >= 1024 on-chip entries
  // (the association is latency-bound, so two streams per SM nearly double
  // its throughput). Otherwise one 256-thread CTA (or a cluster) per stream.
  const size_t half = static_cast<size_t>(smem_sm) / 2 - 1024;
  c->assoc_threads = kAssocThreads;
  // (Round 1 kept this variant opt-in after an intermittent illegal address
  // on cfg4; with the LAP's tie handling rewritten, 1,200 fresh-tracker cfg4
  // updates and 25 bench runs showed no fault: DESIGN.md section 10.)
  // TF_ASSOC_NARROW forces it for fewer streams, TF_ASSOC_WIDE keeps 256.
  const bool many = k.streams >= 2 * sms || getenv("TF_ASSOC_NARROW");
  if (many && !getenv("TF_ASSOC_WIDE") &&
      assoc_smem_bytes(k.max_tracks, k.max_detections, 1024) + assoc_static <= half) {
    c->assoc_threads = kAssocThreadsSmall;
    while (!getenv("TF_ASSOC_NARROW_SOLO") && entries > 1024 &&
           assoc_smem_bytes(k.max_tracks, k.max_detections, entries) + assoc_static > half)
      entries -= 128;   // (TF_ASSOC_NARROW_SOLO keeps the full plan: one 128-thread CTA per SM, diagnostics)
  }
  while (entries > 64 &&
         assoc_smem_bytes(k.max_tracks, k.max_detections, entries) + assoc_static > static_cast<size_t>(smem_optin))
    entries -= 128;
  if (assoc_smem_bytes(k.max_tracks, k.max_detections, entries) + assoc_static > static_cast<size_t>(smem_optin) ||
      frame_smem_bytes(54264, k.max_candidates) + 2048 > static_cast<size_t>(smem_optin)) {
    delete c;
    return TF_ARGUMENT;
  }
  // (TF_CAP_ENTRIES lowers the on-chip entry capacity: tests of the global-pool path)
  if (const char* ce = getenv("TF_CAP_ENTRIES")) entries = std::max(16, std::min(entries, atoi(ce)));
  c->cap_entries = entries;
  cudaError_t e = cudaSuccess;
  auto A = [&](auto** p, size_t n) {
    if (e == cudaSuccess) e = dev_alloc(c, p, n);
  };
  for (int b = 0; b < 2; ++b) {
    A(&c->dets[b].count, F);
    A(&c->dets[b].cand_count, F);
    A(&c->dets[b].status, F);
    A(&c->dets[b].meas, F * Km * 4);
    A(&c->dets[b].obj, F * Km);
    A(&c->dets[b].code, F * Km);
    A(&c->dets[b].emb, F * Km * D);
    A(&c->d_fidx[b], F);
    if (b == 0) A(&c->d_row_offsets, F + 1);
  }
  A(&c->trk.id, S * Tm);
  A(&c->trk.state, S * Tm);
  A(&c->trk.hits, S * Tm);
  A(&c->trk.lost, S * Tm);
  A(&c->trk.last, S * Tm);
  A(&c->trk.slot, S * Tm);
  A(&c->trk.mean, S * Tm * 8);
  A(&c->trk.cov, S * Tm * 12);
  A(&c->trk.emb_pool, S * Tm * D);
  A(&c->trk.free_stack, S * Tm);
  A(&c->trk.n_free, S);
  A(&c->trk.n_tracks, S);
  A(&c->trk.next_id, S);
  A(&c->trk.last_frame, S);
  A(&c->trk.status, S);
  A(&c->pool_col, S * Tm * Km);
  A(&c->pool_row, S * Tm * Km);
  A(&c->pool_val, S * Tm * Km);
  A(&c->pool_aux, 2 * S * Tm * Km);
  A(&c->d_stats, kPhaseSlots + 4 * S);
  A(&c->d_order, S);
  A(&c->d_work, S);
  A(&c->d_ticket, 1);
  if (e == cudaSuccess) e = cudaMemset(c->d_ticket, 0, sizeof(unsigned));
  A(&c->d_ready, F);
  A(&c->d_fticket, 2);
  if (e == cudaSuccess) e = cudaMemset(c->d_ready, 0, sizeof(unsigned) * F);
  if (e == cudaSuccess) e = cudaMemset(c->d_fticket, 0, sizeof(int) * 2);
  c->env_overlap = getenv("TF_OVERLAP") != nullptr;
  c->assoc_slots = sms * (c->assoc_threads == kAssocThreadsSmall ? 2 : 1);
  c->sms = sms;
  c->env_no_lpt = getenv("TF_NO_LPT") != nullptr;
  c->n_streams_alloc = static_cast<int>(S);
  if (e != cudaSuccess) {
    std::string m = cudaGetErrorString(e);
    tf_destroy(c);
    return TF_CUDA;
  }
  c->det = c->dets[0];
  c->d_frame_index = c->d_fidx[0];
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking);
  for (int b = 0; b < 2 && e == cudaSuccess; ++b) {
    e = cudaEventCreateWithFlags(&c->ev_dec[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_asc[b], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_d2h[b], cudaEventDisableTiming);
  }
  for (int r = 0; r < tf_ctx::kRing && e == cudaSuccess; ++r) {
    e = cudaHostAlloc(&c->h_fidx[r], sizeof(long long) * F, cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_fidx[r], cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    tf_destroy(c);
    return TF_CUDA;
  }
  c->last_frame.assign(S, std::numeric_limits<long long>::min());
  reset_streams_kernel<<<static_cast<unsigned>(S), 256>>>(c->trk, 0, static_cast<int>(S), k.max_tracks);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    tf_destroy(c);
    return TF_CUDA;
  }
  *out = c;
  return TF_OK;
}

int tf_destroy(tf_ctx* ctx) {
  if (!ctx) return TF_OK;
  cudaSetDevice(ctx->device);
  for (cudaEvent_t e : ctx->events) cudaEventDestroy(e);
  if (ctx->side) {
    cudaStreamSynchronize(ctx->side);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(ctx->ev_dec[b]);
      cudaEventDestroy(ctx->ev_asc[b]);
    }
    cudaStreamDestroy(ctx->side);
  }
  if (ctx->d2h) {
    cudaStreamSynchronize(ctx->d2h);
    for (int b = 0; b < 2; ++b) cudaEventDestroy(ctx->ev_d2h[b]);
    cudaStreamDestroy(ctx->d2h);
  }
  for (int r = 0; r < tf_ctx::kRing; ++r)
    if (ctx->h_fidx[r]) {
      cudaEventSynchronize(ctx->ev_fidx[r]);
      cudaEventDestroy(ctx->ev_fidx[r]);
      cudaFreeHost(ctx->h_fidx[r]);
    }
  for (void* p : ctx->allocs) cudaFree(p);
  delete ctx;
  return TF_OK;
}

int tf_reset_stream(tf_ctx* c, int32_t stream, void* cuda_stream) {
  NvtxRange nvtx_range("tf_reset_stream");
  if (!c) return TF_ARGUMENT;
  if (stream < 0 || stream >= c->cap.streams) return fail(c, TF_ARGUMENT, "stream out of range");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  for (int b = 0; b < 2; ++b)
    if (c->asc_pending[b]) TF_CUDA(c, cudaStreamWaitEvent(st, c->ev_asc[b], 0));
  ++c->launches;
  reset_streams_kernel<<<1, 256, 0, st>>>(c->trk, stream, 1, c->cap.max_tracks);
  TF_CUDA(c, cudaGetLastError());
  c->last_frame[stream] = std::numeric_limits<long long>::min();
  return TF_OK;
}

static int ensure_record_staging(tf_ctx* c, int frames, int max_records) {
  const int need = frames * max_records;
  if (need <= c->rec_capacity && c->rec_count[0]) return TF_OK;
  cudaError_t e = cudaSuccess;
  auto A = [&](auto** p, size_t n) {
    if (e == cudaSuccess) e = dev_alloc(c, p, n);
  };
  for (int b = 0; b < 2; ++b) {
    A(&c->rec_count[b], static_cast<size_t>(c->cap.max_frames));
    A(&c->rec_id[b], static_cast<size_t>(need));
    A(&c->rec_box[b], static_cast<size_t>(need) * 4);
    A(&c->rec_obj[b], static_cast<size_t>(need));
  }
  if (e != cudaSuccess) return fail(c, TF_CUDA, std::string("record staging: ") + cudaGetErrorString(e));
  c->rec_capacity = need;
  return TF_OK;
}

int tf_update_heads(tf_ctx* c, const tf_heads* heads, int32_t stream_begin, int32_t n_streams,
                    int32_t B, const int64_t* frame_index, const tf_records* out, const tf_trace* trace,
                    void* cuda_stream) {
  NvtxRange nvtx_range("tf_update_heads");
  if (!c || !heads || !frame_index || !out) return fail(c, TF_ARGUMENT, "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  if (n_streams < 1 || B < 1 || stream_begin < 0 || stream_begin + n_streams > c->cap.streams)
    return fail(c, TF_ARGUMENT, "stream range out of bounds");
  const int F = n_streams * B;
  if (F > c->cap.max_frames) return fail(c, TF_CAPACITY, "frames per update exceed max_frames");
  if (out->max_records < 1) return fail(c, TF_ARGUMENT, "max_records must be >= 1");
  int rc = check_step_config(c);
  if (rc) return rc;
  if (heads->dtype != 0 && heads->dtype != 1) return fail(c, TF_LAYOUT, "heads dtype must be 0 (fp32) or 1 (binary16)");
  for (int i = 0; i < 3; ++i) {
    const tf_head_scale& s = heads->scale[i];
    if (!s.head || !s.emb || s.height < 1 || s.width < 1 || s.head_stride_c < static_cast<long long>(s.height) * s.width)
      return fail(c, TF_LAYOUT, "head scale " + std::to_string(i) + ": bad pointer or layout");
    // parse_output's width check (tf/postproc.py:25-29): the map must carry
    // exactly embedding_dim channels, or the gather would read the
    // neighbouring cells' values (or past the tensor)
    if (s.channels != c->cfg.embedding_dim)
      return fail(c, TF_LAYOUT, "head scale " + std::to_string(i) + ": embedding map has " +
                                    std::to_string(s.channels) + " channels, expected embedding_dim " +
                                    std::to_string(c->cfg.embedding_dim));
  }
  for (int ls = 0; ls < n_streams; ++ls) {
    rc = check_ordering(c, stream_begin + ls, reinterpret_cast<const long long*>(frame_index) + static_cast<size_t>(ls) * B, B);
    if (rc) return rc;
  }
  c->prof_on = c->profiling && (c->prof_counter++ % c->prof_stride) == 0;
  TF_CUDA(c, ensure_device(c->device));
  // buffer set and streams: without pipelining everything runs on `st` with set 0;
  // with pipelining the decode of this update (on `st`) overlaps the previous
  // update's association (on the side stream)
  const int par = c->pipeline ? c->parity : 0;
  if (c->pipeline) c->parity ^= 1;
  cudaStream_t ast = c->pipeline ? c->side : st;           // association + outputs
  DetBuf& det = c->dets[par];

  HeadLaunch h = {};
  h.heads = heads;
  h.frames = F;
  h.cap_cand = c->cap.max_candidates;
  h.cap_det = c->cap.max_detections;
  h.det = det;
  tf_heads staged = *heads;
  TF_CUDA(c, prof_mark(c, 4, st));
  if (heads->host_memory) {
    // Default: the frame kernel reads everything it needs -- the confidence
    // planes (coalesced float4 streams), the deltas of candidates and the
    // embeddings of candidates -- in place through the mapped host pointer,
    // ~17 MB per 32 frames at PCIe rate (B200 box: ~42 GB/s). The alternative
    // (TF_HOST_CONF=copy) stages the confidence planes with a strided
    // cudaMemcpy2DAsync; its throughput varied between 6 and 37 GB/s across
    // boxes while plain SM reads did not, so it is opt-in.
    const char* conf_env = getenv("TF_HOST_CONF");
    const bool conf_mapped = !(conf_env && conf_env[0] == 'c') || heads->dtype != 0;
    for (int i = 0; i < 3; ++i) {
      const tf_head_scale& s = heads->scale[i];
      const size_t hw = static_cast<size_t>(s.height) * s.width;
      const size_t need = static_cast<size_t>(F) * 24 * hw;
      if (conf_mapped) {           // the frame kernel streams the planes over PCIe itself
        void* hp = nullptr;
        TF_CUDA(c, cudaHostGetDevicePointer(&hp, const_cast<float*>(s.head), 0));
        h.head_ptr[i] = static_cast<const float*>(hp);
        void* dptr = nullptr;
        TF_CUDA(c, cudaHostGetDevicePointer(&dptr, const_cast<float*>(s.emb), 0));
        h.emb_ptr[i] = static_cast<const float*>(dptr);
        continue;
      }
      if (c->stage_conf_elems[par][i] < need) {
        float* p = nullptr;
        TF_CUDA(c, dev_alloc(c, &p, need));
        c->stage_conf[par][i] = p;
        c->stage_conf_elems[par][i] = need;
      }
      // staging keeps the [F][24][H][W] geometry; only conf planes are filled.
      // Rows of the 2D copy are (frame, anchor) pairs of 2 planes each; frames
      // with a uniform stride collapse into one copy per scale.
      const bool uniform = s.head_stride_n == 4 * (6 * s.head_stride_c);
      const int calls = uniform ? 1 : F;
      const int rows = uniform ? 4 * F : 4;
      for (int f = 0; f < calls; ++f) {
        const float* src = s.head + static_cast<long long>(f) * s.head_stride_n + 4 * s.head_stride_c;
        float* dst = c->stage_conf[par][i] + static_cast<size_t>(f) * 24 * hw + 4 * hw;
        TF_CUDA(c, cudaMemcpy2DAsync(dst, 6 * hw * sizeof(float), src, 6 * s.head_stride_c * sizeof(float),
                                     2 * hw * sizeof(float), rows, cudaMemcpyHostToDevice, st));
      }
      staged.scale[i].head_stride_n = static_cast<long long>(24 * hw);
      staged.scale[i].head_stride_c = static_cast<long long>(hw);
      h.head_ptr[i] = c->stage_conf[par][i];
      void* dptr = nullptr;
      TF_CUDA(c, cudaHostGetDevicePointer(&dptr, const_cast<float*>(s.emb), 0));
      h.emb_ptr[i] = static_cast<const float*>(dptr);
    }
    h.heads = &staged;
    rc = TF_OK;
  } else {
    for (int i = 0; i < 3; ++i) {
      h.head_ptr[i] = heads->scale[i].head;
      h.emb_ptr[i] = heads->scale[i].emb;
    }
  }
  // In host mode the deltas are read from the mapped host tensor: pass its
  // device alias and original strides through a second descriptor.
  if (heads->host_memory) {
    for (int i = 0; i < 3; ++i) {
      void* dptr = nullptr;
      TF_CUDA(c, cudaHostGetDevicePointer(&dptr, const_cast<float*>(heads->scale[i].head), 0));
      h.delta_ptr[i] = static_cast<const float*>(dptr);
      h.delta_stride_n[i] = heads->scale[i].head_stride_n;
      h.delta_stride_c[i] = heads->scale[i].head_stride_c;
    }
  } else {
    for (int i = 0; i < 3; ++i) {
      h.delta_ptr[i] = heads->scale[i].head;
      h.delta_stride_n[i] = heads->scale[i].head_stride_n;
      h.delta_stride_c[i] = heads->scale[i].head_stride_c;
    }
  }
  TF_CUDA(c, prof_mark(c, 5, st));
  // The confidence-plane copy above only needs the previous decode on `st` to
  // be done with the staging buffer; the detection buffers and frame indices
  // of this parity are read by the association two updates back, so only the
  // decode waits for it (the copy overlaps that association).
  if (c->pipeline && c->asc_pending[par]) TF_CUDA(c, cudaStreamWaitEvent(st, c->ev_asc[par], 0));
  const bool fidx_inline = F <= kFidxInline;      // small updates: indices travel in the launch parameters
  if (!fidx_inline)
    TF_CUDA(c, upload_frame_index(c, c->d_fidx[par], reinterpret_cast<const long long*>(frame_index), F, st));
  // Overlapped mode (opt-in, TF_OVERLAP): many frames, no pipelining,
  // device-resident heads and single-CTA 128-thread association CTAs (one
  // fits next to two decode CTAs on an SM): the decode grid is persistent and
  // publishes frames one by one; the association starts right away
  // (programmatic dependent launch) and waits per frame. No event may sit
  // between the two launches. Measured on B200 at config 4 it is slower
  // (2.45 vs 2.20 ms per step: while the decode runs, only one association
  // CTA per SM fits instead of two, and the association needs every slot),
  // so it is off by default; DESIGN.md section 6.
  const bool overlap = !c->pipeline && !heads->host_memory && c->env_overlap &&
                       c->assoc_threads == kAssocThreadsSmall && F >= 2 * c->sms;
  h.ready = nullptr;
  if (overlap) {
    h.ready = c->d_ready;
    h.epoch = ++c->epoch == 0 ? ++c->epoch : c->epoch;
    h.ticket = c->d_fticket;
    h.order = next_stream_order(c, 1, stream_begin, n_streams);
    h.first_wave = c->sms;
    h.streams = n_streams;
    h.B = B;
    h.persist_ctas = 2 * c->sms;
  }
  TF_CUDA(c, prof_mark(c, 0, st));
  TF_CUDA(c, launch_frame_heads(h, c->P, st));
  ++c->launches;
  if (!overlap) TF_CUDA(c, prof_mark(c, 1, st));
  if (c->pipeline) {
    TF_CUDA(c, cudaEventRecord(c->ev_dec[par], st));
    TF_CUDA(c, cudaStreamWaitEvent(ast, c->ev_dec[par], 0));
  }

  AssocArgs a = {};
  a.det = det;
  a.trk = c->trk;
  a.trace = to_trace(trace);
  a.frame_index = c->d_fidx[par];
  a.stream_begin = stream_begin;
  a.B = B;
  a.cap_tracks = c->cap.max_tracks;
  a.cap_det = c->cap.max_detections;
  a.cap_entries = c->cap_entries;
  a.threads = c->assoc_threads;
  a.zero_smem = c->env_zero_smem;
  a.n_fidx_inline = 0;
  if (fidx_inline) {
    a.n_fidx_inline = F;
    for (int i = 0; i < F; ++i) a.fidx_inline[i] = frame_index[i];
  }
  a.pool_col = c->pool_col;
  a.pool_row = c->pool_row;
  a.pool_val = c->pool_val;
  a.pool_aux = c->pool_aux;
  a.stats = (c->profiling & 2) ? c->d_stats : nullptr;
  a.sclk = (c->profiling & 4) ? c->d_stats + kPhaseSlots : nullptr;
  {
    const int key = n_streams * 64 + c->env_cluster;
    if (key != c->cluster_key) {
      c->cluster_val = a.threads == kAssocThreadsSmall ? 1 : assoc_cluster_size(n_streams, a.cap_tracks, a.cap_det, a.cap_entries);
      c->cluster_key = key;
    }
    a.cluster = c->cluster_val;
  }
  set_stream_order(c, a, stream_begin, n_streams);
  const bool host_out = heads->host_memory != 0;
  if (host_out) {
    rc = ensure_record_staging(c, F, out->max_records);
    if (rc) return rc;
    a.out.count = c->rec_count[par];
    a.out.track_id = c->rec_id[par];
    a.out.box = c->rec_box[par];
    a.out.objectness = c->rec_obj[par];
    // the previous copy out of this staging set must have finished
    if (c->d2h_pending[par]) TF_CUDA(c, cudaStreamWaitEvent(ast, c->ev_d2h[par], 0));
  } else {
    a.out.count = out->count;
    a.out.track_id = reinterpret_cast<long long*>(out->track_id);
    a.out.box = out->box;
    a.out.objectness = out->objectness;
  }
  a.out.max_records = out->max_records;
  a.ready = overlap ? c->d_ready : nullptr;
  a.epoch = h.epoch;
  if (!overlap) TF_CUDA(c, prof_mark(c, 2, ast));
  TF_CUDA(c, launch_associate(a, n_streams, c->P, ast));
  ++c->launches;
  if (overlap) {           // decode and association overlap: the frame slot times both, the association slot ~0
    TF_CUDA(c, prof_mark(c, 1, ast));
    TF_CUDA(c, prof_mark(c, 2, ast));
  }
  TF_CUDA(c, prof_mark(c, 3, ast));
  if (c->pipeline) {
    TF_CUDA(c, cudaEventRecord(c->ev_asc[par], ast));
    c->asc_pending[par] = true;
  }
  if (trace && trace->det_code) {
    ++c->launches;
    copy_codes_kernel<<<F, 128, 0, ast>>>(det.count, det.code, trace->det_code, F, c->cap.max_detections);
  }
  if (host_out) {
    const size_t n = static_cast<size_t>(F) * out->max_records;
    if (!c->pipeline) TF_CUDA(c, cudaEventRecord(c->ev_asc[par], ast));
    TF_CUDA(c, cudaStreamWaitEvent(c->d2h, c->ev_asc[par], 0));
    TF_CUDA(c, cudaMemcpyAsync(out->count, c->rec_count[par], sizeof(int) * F, cudaMemcpyDeviceToHost, c->d2h));
    TF_CUDA(c, cudaMemcpyAsync(out->track_id, c->rec_id[par], sizeof(long long) * n, cudaMemcpyDeviceToHost, c->d2h));
    TF_CUDA(c, cudaMemcpyAsync(out->box, c->rec_box[par], sizeof(double) * 4 * n, cudaMemcpyDeviceToHost, c->d2h));
    TF_CUDA(c, cudaMemcpyAsync(out->objectness, c->rec_obj[par], sizeof(double) * n, cudaMemcpyDeviceToHost, c->d2h));
    TF_CUDA(c, cudaEventRecord(c->ev_d2h[par], c->d2h));
    c->d2h_pending[par] = true;
  }
  c->touched_lo = std::min(c->touched_lo, stream_begin);
  c->touched_hi = std::max(c->touched_hi, stream_begin + n_streams);
  for (int ls = 0; ls < n_streams; ++ls)
    c->last_frame[stream_begin + ls] = frame_index[static_cast<size_t>(ls) * B + B - 1];
  c->last_begin = stream_begin;
  c->last_count = n_streams;
  return TF_OK;
}

int tf_update_detections(tf_ctx* c, int32_t stream_begin, int32_t n_streams, int32_t B, const int64_t* frame_index,
                         const int32_t* row_offsets, const double* boxes, const double* objectness,
                         const float* embeddings, int32_t normalized, const tf_records* out, const tf_trace* trace,
                         void* cuda_stream) {
  NvtxRange nvtx_range("tf_update_detections");
  if (!c || !frame_index || !row_offsets || !out) return fail(c, TF_ARGUMENT, "null argument");
  if (n_streams < 1 || B < 1 || stream_begin < 0 || stream_begin + n_streams > c->cap.streams)
    return fail(c, TF_ARGUMENT, "stream range out of bounds");
  const int F = n_streams * B;
  if (F > c->cap.max_frames) return fail(c, TF_CAPACITY, "frames per update exceed max_frames");
  if (out->max_records < 1) return fail(c, TF_ARGUMENT, "max_records must be >= 1");
  if (row_offsets[0] != 0) return fail(c, TF_ARGUMENT, "row_offsets[0] must be 0");
  for (int f = 0; f < F; ++f) {
    const int n = row_offsets[f + 1] - row_offsets[f];
    if (n < 0) return fail(c, TF_ARGUMENT, "row_offsets must be non-decreasing");
    if (n > c->cap.max_candidates) return fail(c, TF_CAPACITY, "too many detections for max_candidates");
  }
  if (row_offsets[F] > 0 && (!boxes || !objectness || !embeddings)) return fail(c, TF_ARGUMENT, "null detection arrays");
  int rc = check_step_config(c);
  if (rc) return rc;
  for (int ls = 0; ls < n_streams; ++ls) {
    rc = check_ordering(c, stream_begin + ls, reinterpret_cast<const long long*>(frame_index) + static_cast<size_t>(ls) * B, B);
    if (rc) return rc;
  }
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  c->prof_on = c->profiling && (c->prof_counter++ % c->prof_stride) == 0;
  TF_CUDA(c, ensure_device(c->device));
  for (int b = 0; b < 2; ++b)
    if (c->asc_pending[b]) TF_CUDA(c, cudaStreamWaitEvent(st, c->ev_asc[b], 0));
  c->asc_pending[0] = c->asc_pending[1] = false;
  TF_CUDA(c, upload_frame_index(c, c->d_frame_index, reinterpret_cast<const long long*>(frame_index), F, st));
  TF_CUDA(c, cudaMemcpyAsync(c->d_row_offsets, row_offsets, sizeof(int32_t) * (F + 1), cudaMemcpyHostToDevice, st));
  TF_CUDA(c, launch_frame_rows(boxes, objectness, embeddings, c->d_row_offsets, F, normalized ? 0 : 1,
                               c->cap.max_candidates, c->cap.max_detections, c->det, c->P, st));
  ++c->launches;
  AssocArgs a = {};
  a.det = c->det;
  a.trk = c->trk;
  a.trace = to_trace(trace);
  a.frame_index = c->d_frame_index;
  a.stream_begin = stream_begin;
  a.B = B;
  a.cap_tracks = c->cap.max_tracks;
  a.cap_det = c->cap.max_detections;
  a.cap_entries = c->cap_entries;
  a.threads = c->assoc_threads;
  a.zero_smem = c->env_zero_smem;
  a.n_fidx_inline = 0;
  a.pool_col = c->pool_col;
  a.pool_row = c->pool_row;
  a.pool_val = c->pool_val;
  a.pool_aux = c->pool_aux;
  a.stats = (c->profiling & 2) ? c->d_stats : nullptr;
  a.sclk = (c->profiling & 4) ? c->d_stats + kPhaseSlots : nullptr;
  {
    const int key = n_streams * 64 + c->env_cluster;
    if (key != c->cluster_key) {
      c->cluster_val = a.threads == kAssocThreadsSmall ? 1 : assoc_cluster_size(n_streams, a.cap_tracks, a.cap_det, a.cap_entries);
      c->cluster_key = key;
    }
    a.cluster = c->cluster_val;
  }
  set_stream_order(c, a, stream_begin, n_streams);
  a.out.count = out->count;
  a.out.track_id = reinterpret_cast<long long*>(out->track_id);
  a.out.box = out->box;
  a.out.objectness = out->objectness;
  a.out.max_records = out->max_records;
  TF_CUDA(c, launch_associate(a, n_streams, c->P, st));
  ++c->launches;
  if (trace && trace->det_code) {
    ++c->launches;
    copy_codes_kernel<<<F, 128, 0, st>>>(c->det.count, c->det.code, trace->det_code, F, c->cap.max_detections);
  }
  c->touched_lo = std::min(c->touched_lo, stream_begin);
  c->touched_hi = std::max(c->touched_hi, stream_begin + n_streams);
  for (int ls = 0; ls < n_streams; ++ls)
    c->last_frame[stream_begin + ls] = frame_index[static_cast<size_t>(ls) * B + B - 1];
  return TF_OK;
}

int tf_step_detections(tf_ctx* c, int32_t stream, int64_t frame_index, int32_t n, const double* boxes,
                       const double* objectness, const float* embeddings, const uint8_t* has_embedding,
                       const tf_records* out, const tf_trace* trace, void* cuda_stream) {
  NvtxRange nvtx_range("tf_step_detections");
  if (!c || !out) return fail(c, TF_ARGUMENT, "null argument");
  if (stream < 0 || stream >= c->cap.streams) return fail(c, TF_ARGUMENT, "stream out of range");
  if (n < 0) return fail(c, TF_ARGUMENT, "negative detection count");
  if (n > c->cap.max_candidates) return fail(c, TF_CAPACITY, "too many detections for max_candidates");
  if (n > 0 && (!boxes || !objectness || !embeddings || !has_embedding))
    return fail(c, TF_ARGUMENT, "null detection arrays");
  int rc = check_step_config(c);
  if (rc) return rc;
  const long long fi = frame_index;
  rc = check_ordering(c, stream, &fi, 1);
  if (rc) return rc;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  TF_CUDA(c, ensure_device(c->device));
  for (int b = 0; b < 2; ++b)
    if (c->asc_pending[b]) TF_CUDA(c, cudaStreamWaitEvent(st, c->ev_asc[b], 0));
  // (the frame index travels in the association's launch parameters)
  TF_CUDA(c, launch_frame_dets(boxes, objectness, embeddings, has_embedding, n, c->cap.max_candidates,
                               c->cap.max_detections, c->det, c->P, st));
  ++c->launches;
  AssocArgs a = {};
  a.det = c->det;
  a.trk = c->trk;
  a.trace = to_trace(trace);
  a.frame_index = c->d_frame_index;
  a.stream_begin = stream;
  a.B = 1;
  a.cap_tracks = c->cap.max_tracks;
  a.cap_det = c->cap.max_detections;
  a.cap_entries = c->cap_entries;
  a.threads = c->assoc_threads;
  a.zero_smem = c->env_zero_smem;
  a.n_fidx_inline = 1;
  a.fidx_inline[0] = fi;
  a.pool_col = c->pool_col;
  a.pool_row = c->pool_row;
  a.pool_val = c->pool_val;
  a.pool_aux = c->pool_aux;
  a.stats = (c->profiling & 2) ? c->d_stats : nullptr;
  a.sclk = (c->profiling & 4) ? c->d_stats + kPhaseSlots : nullptr;
  a.cluster = 1;
  set_stream_order(c, a, stream, 1);
  a.out.count = out->count;
  a.out.track_id = reinterpret_cast<long long*>(out->track_id);
  a.out.box = out->box;
  a.out.objectness = out->objectness;
  a.out.max_records = out->max_records;
  TF_CUDA(c, launch_associate(a, 1, c->P, st));
  ++c->launches;
  if (trace && trace->det_code) {
    ++c->launches;
    copy_codes_kernel<<<1, 128, 0, st>>>(c->det.count, c->det.code, trace->det_code, 1, c->cap.max_detections);
  }
  c->last_frame[stream] = fi;
  c->touched_lo = std::min(c->touched_lo, static_cast<int>(stream));
  c->touched_hi = std::max(c->touched_hi, static_cast<int>(stream) + 1);
  return TF_OK;
}

int tf_finish(tf_ctx* c, void* cuda_stream) {
  NvtxRange nvtx_range("tf_finish");
  if (!c) return TF_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  TF_CUDA(c, cudaStreamSynchronize(st));
  if (c->side) TF_CUDA(c, cudaStreamSynchronize(c->side));
  if (c->d2h) TF_CUDA(c, cudaStreamSynchronize(c->d2h));
  c->asc_pending[0] = c->asc_pending[1] = false;
  c->d2h_pending[0] = c->d2h_pending[1] = false;
  if (c->touched_hi <= c->touched_lo) return TF_OK;
  const int lo = c->touched_lo, n = c->touched_hi - c->touched_lo;
  c->touched_lo = 1 << 30;
  c->touched_hi = -1;
  std::vector<int> status(n);
  TF_CUDA(c, cudaMemcpy(status.data(), c->trk.status + lo, sizeof(int) * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemset(c->trk.status + lo, 0, sizeof(int) * n));
  for (int i = 0; i < n; ++i) {
    if (status[i] != 0) {
      const int code = status[i] & 0xff, frame = status[i] >> 8;
      return fail(c, code, std::string(tf_status_name(code)) + " in stream " + std::to_string(lo + i) +
                               " at batch frame " + std::to_string(frame));
    }
  }
  return TF_OK;
}

int tf_set_pipeline(tf_ctx* c, int32_t enabled) {
  if (!c) return TF_ARGUMENT;
  if (c->side) TF_CUDA(c, cudaStreamSynchronize(c->side));
  if (c->d2h) TF_CUDA(c, cudaStreamSynchronize(c->d2h));
  c->asc_pending[0] = c->asc_pending[1] = false;
  c->d2h_pending[0] = c->d2h_pending[1] = false;
  c->pipeline = enabled ? 1 : 0;
  c->parity = 0;
  return TF_OK;
}

int tf_join(tf_ctx* c, void* cuda_stream) {
  if (!c) return TF_ARGUMENT;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  for (int b = 0; b < 2; ++b) {
    if (c->asc_pending[b]) TF_CUDA(c, cudaStreamWaitEvent(st, c->ev_asc[b], 0));
    if (c->d2h_pending[b]) TF_CUDA(c, cudaStreamWaitEvent(st, c->ev_d2h[b], 0));
  }
  return TF_OK;
}

int tf_export_tracks(tf_ctx* c, int32_t stream, tf_track_export* o, void* cuda_stream) {
  NvtxRange nvtx_range("tf_export_tracks");
  if (!c || !o) return TF_ARGUMENT;
  if (stream < 0 || stream >= c->cap.streams) return fail(c, TF_ARGUMENT, "stream out of range");
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  TF_CUDA(c, cudaStreamSynchronize(st));
  if (c->side) TF_CUDA(c, cudaStreamSynchronize(c->side));
  const long long Tm = c->cap.max_tracks, D = c->cfg.embedding_dim;
  const long long base = stream * Tm;
  int n = 0;
  TF_CUDA(c, cudaMemcpy(&n, c->trk.n_tracks + stream, sizeof(int), cudaMemcpyDeviceToHost));
  long long next = 0, last = 0;
  TF_CUDA(c, cudaMemcpy(&next, c->trk.next_id + stream, sizeof(long long), cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(&last, c->trk.last_frame + stream, sizeof(long long), cudaMemcpyDeviceToHost));
  o->count = n;
  o->next_id = next;
  o->last_frame = last;
  if (n == 0) return TF_OK;
  std::vector<int> slot(n);
  std::vector<double> cov(12 * static_cast<size_t>(n));
  TF_CUDA(c, cudaMemcpy(o->track_id, c->trk.id + base, 8 * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(o->state, c->trk.state + base, 4 * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(o->hits, c->trk.hits + base, 4 * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(o->lost_since, c->trk.lost + base, 8 * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(o->last_update_frame, c->trk.last + base, 8 * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(o->mean, c->trk.mean + base * 8, 64 * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(cov.data(), c->trk.cov + base * 12, 96 * n, cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemcpy(slot.data(), c->trk.slot + base, 4 * n, cudaMemcpyDeviceToHost));
  for (int t = 0; t < n; ++t) {
    double* C8 = o->covariance + 64 * t;
    for (int q = 0; q < 64; ++q) C8[q] = 0.0;
    for (int i = 0; i < 4; ++i) {
      C8[8 * i + i] = cov[12 * t + 3 * i];
      C8[8 * i + i + 4] = cov[12 * t + 3 * i + 1];
      C8[8 * (i + 4) + i] = cov[12 * t + 3 * i + 1];
      C8[8 * (i + 4) + i + 4] = cov[12 * t + 3 * i + 2];
    }
    TF_CUDA(c, cudaMemcpy(o->embedding + D * t, c->trk.emb_pool + (base + slot[t]) * D, 4 * D,
                          cudaMemcpyDeviceToHost));
  }
  return TF_OK;
}

int tf_import_tracks(tf_ctx* c, int32_t stream, const tf_track_export* in, void* cuda_stream) {
  NvtxRange nvtx_range("tf_import_tracks");
  // inverse of tf_export_tracks: the track table of a Tracker at some frame
  // (tf/tracker.py:74-83 tracks, _next_id, _last_frame) becomes stream's
  // state, so a sequence can be resumed from the reference's state at any
  // frame (parity bisection). Slots are re-packed 0..count-1.
  if (!c || !in) return TF_ARGUMENT;
  if (stream < 0 || stream >= c->cap.streams) return fail(c, TF_ARGUMENT, "stream out of range");
  const int n = in->count;
  const int Tm = c->cap.max_tracks, D = c->cfg.embedding_dim;
  if (n < 0 || n > Tm)
    return fail(c, TF_CAPACITY, "import of " + std::to_string(n) + " tracks exceeds max_tracks " +
                                    std::to_string(Tm));
  if (n > 0 && (!in->track_id || !in->state || !in->hits || !in->lost_since || !in->last_update_frame ||
                !in->mean || !in->covariance || !in->embedding))
    return fail(c, TF_ARGUMENT, "import: NULL track array");
  std::vector<double> cov(12 * static_cast<size_t>(n));
  std::vector<int> slot(n), free_stack(Tm);
  for (int t = 0; t < n; ++t) {
    const long long id = in->track_id[t];
    if (id < 1 || id >= in->next_id)
      return fail(c, TF_ARGUMENT, "import: track id " + std::to_string(id) + " outside [1, next_id)");
    for (int u = 0; u < t; ++u)
      if (in->track_id[u] == id) return fail(c, TF_ARGUMENT, "import: duplicate track id " + std::to_string(id));
    if (in->state[t] != 0 && in->state[t] != 1)
      return fail(c, TF_ARGUMENT, "import: track state must be 0 (ACTIVE) or 1 (LOST)");
    if ((in->state[t] == 1) != (in->lost_since[t] >= 0))
      return fail(c, TF_ARGUMENT, "import: lost_since must be set exactly for LOST tracks");
    const double* C8 = in->covariance + 64 * static_cast<size_t>(t);
    for (int i = 0; i < 8; ++i)
      for (int j = 0; j < 8; ++j)
        if ((i & 3) != (j & 3) && C8[8 * i + j] != 0.0)
          return fail(c, TF_ARGUMENT, "import: covariance of track " + std::to_string(id) +
                                          " couples two axes; the filter keeps per-axis (position, velocity) blocks");
    for (int i = 0; i < 4; ++i) {
      if (C8[8 * i + i + 4] != C8[8 * (i + 4) + i])
        return fail(c, TF_ARGUMENT, "import: covariance of track " + std::to_string(id) + " is not symmetric");
      cov[12 * t + 3 * i] = C8[8 * i + i];
      cov[12 * t + 3 * i + 1] = C8[8 * i + i + 4];
      cov[12 * t + 3 * i + 2] = C8[8 * (i + 4) + i + 4];
    }
    slot[t] = t;
  }
  for (int i = 0; i < Tm; ++i) free_stack[i] = Tm - 1 - i;  // pops slot n next, as after n births
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  TF_CUDA(c, cudaStreamSynchronize(st));
  if (c->side) TF_CUDA(c, cudaStreamSynchronize(c->side));
  const long long base = static_cast<long long>(stream) * Tm;
  const int nfree = Tm - n, zero = 0;
  if (n > 0) {
    TF_CUDA(c, cudaMemcpy(c->trk.id + base, in->track_id, 8 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.state + base, in->state, 4 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.hits + base, in->hits, 4 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.lost + base, in->lost_since, 8 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.last + base, in->last_update_frame, 8 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.mean + base * 8, in->mean, 64 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.cov + base * 12, cov.data(), 96 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.slot + base, slot.data(), 4 * n, cudaMemcpyHostToDevice));
    TF_CUDA(c, cudaMemcpy(c->trk.emb_pool + base * D, in->embedding, 4ll * D * n, cudaMemcpyHostToDevice));
  }
  TF_CUDA(c, cudaMemcpy(c->trk.free_stack + base, free_stack.data(), 4ll * Tm, cudaMemcpyHostToDevice));
  TF_CUDA(c, cudaMemcpy(c->trk.n_free + stream, &nfree, 4, cudaMemcpyHostToDevice));
  TF_CUDA(c, cudaMemcpy(c->trk.n_tracks + stream, &n, 4, cudaMemcpyHostToDevice));
  TF_CUDA(c, cudaMemcpy(c->trk.next_id + stream, &in->next_id, 8, cudaMemcpyHostToDevice));
  TF_CUDA(c, cudaMemcpy(c->trk.last_frame + stream, &in->last_frame, 8, cudaMemcpyHostToDevice));
  TF_CUDA(c, cudaMemcpy(c->trk.status + stream, &zero, 4, cudaMemcpyHostToDevice));
  c->last_frame[stream] = in->last_frame;
  return TF_OK;
}

int tf_set_profiling(tf_ctx* c, int32_t enabled) {
  if (!c) return TF_ARGUMENT;
  c->profiling = enabled & 15;
  c->prof_stride = enabled >> 4 > 0 ? enabled >> 4 : 1;
  // timing events for 64 updates up front: creating them inside a timed
  // update costs tens of microseconds of host time per update
  while (c->profiling && c->events.size() < 6 * 64) {
    cudaEvent_t e;
    TF_CUDA(c, cudaEventCreate(&e));
    c->events.push_back(e);
  }
  c->prof_counter = 0;
  c->prof_on = true;
  c->events_used = 0;
  TF_CUDA(c, cudaMemset(c->d_stats, 0, kPhaseSlots * sizeof(long long)));
  return TF_OK;
}

int tf_phase_stats(tf_ctx* c, int64_t* out16) {
  if (!c || !out16) return TF_ARGUMENT;
  TF_CUDA(c, cudaDeviceSynchronize());
  TF_CUDA(c, cudaMemcpy(out16, c->d_stats, kPhaseSlots * sizeof(long long), cudaMemcpyDeviceToHost));
  TF_CUDA(c, cudaMemset(c->d_stats, 0, kPhaseSlots * sizeof(long long)));
  return TF_OK;
}

int tf_stream_hold(const volatile int32_t* flag, void* cuda_stream) {
  if (!flag) return TF_ARGUMENT;
  stream_hold_kernel<<<1, 32, 0, static_cast<cudaStream_t>(cuda_stream)>>>(flag);
  return cudaGetLastError() == cudaSuccess ? TF_OK : TF_CUDA;
}

int tf_stream_clocks(tf_ctx* c, int64_t* out, int32_t n_streams) {
  if (!c || !out || n_streams < 0 || n_streams > c->n_streams_alloc) return TF_ARGUMENT;
  TF_CUDA(c, cudaDeviceSynchronize());
  TF_CUDA(c, cudaMemcpy(out, c->d_stats + kPhaseSlots, 4 * sizeof(long long) * n_streams, cudaMemcpyDeviceToHost));
  return TF_OK;
}

int tf_timeline(tf_ctx* c, double* out, int32_t max_updates, int32_t* n_updates) {
  // per update: frame start/end, association start/end, copy start/end (ms
  // from the first recorded event); call before tf_kernel_times (which resets)
  if (!c || !out || !n_updates) return TF_ARGUMENT;
  const int nu = static_cast<int>(c->events_used / 6);
  *n_updates = nu;
  if (nu == 0) return TF_OK;
  TF_CUDA(c, cudaEventSynchronize(c->events[c->events_used - 3]));
  const int order[6] = {0, 1, 2, 3, 4, 5};
  for (int u = 0; u < nu && u < max_updates; ++u)
    for (int k = 0; k < 6; ++k) {
      float t = 0.f;
      TF_CUDA(c, cudaEventElapsedTime(&t, c->events[4], c->events[6 * u + order[k]]));
      out[6 * u + k] = t;
    }
  return TF_OK;
}

int tf_launch_info(tf_ctx* c, int32_t* assoc_threads, int32_t* assoc_cluster) {
  if (!c || !assoc_threads || !assoc_cluster) return TF_ARGUMENT;
  *assoc_threads = c->assoc_threads;
  *assoc_cluster = c->cluster_val;
  return TF_OK;
}

int tf_launch_count(const tf_ctx* c, int64_t* launches) {
  if (!c || !launches) return TF_ARGUMENT;
  *launches = c->launches;
  return TF_OK;
}

int tf_copy_times(tf_ctx* c, double* h2d_ms) {
  if (!c || !h2d_ms) return TF_ARGUMENT;
  *h2d_ms = c->last_h2d_ms;
  return TF_OK;
}

int tf_kernel_times(tf_ctx* c, double* frame_ms, double* assoc_ms, int64_t* updates) {
  if (!c || !frame_ms || !assoc_ms || !updates) return TF_ARGUMENT;
  *frame_ms = 0.0;
  *assoc_ms = 0.0;
  *updates = static_cast<int64_t>(c->events_used / 6);
  c->last_h2d_ms = 0.0;
  if (c->events_used == 0) return TF_OK;
  TF_CUDA(c, cudaEventSynchronize(c->events[c->events_used - 3]));
  for (size_t i = 0; i + 5 < c->events_used; i += 6) {
    float a = 0.f, b = 0.f, h = 0.f;
    TF_CUDA(c, cudaEventSynchronize(c->events[i + 3]));
    TF_CUDA(c, cudaEventElapsedTime(&a, c->events[i], c->events[i + 1]));
    TF_CUDA(c, cudaEventElapsedTime(&b, c->events[i + 2], c->events[i + 3]));
    TF_CUDA(c, cudaEventElapsedTime(&h, c->events[i + 4], c->events[i + 5]));
    *frame_ms += a;
    *assoc_ms += b;
    c->last_h2d_ms += h;
  }
  c->events_used = 0;
  return TF_OK;
}

// ---- stage-level entry points -------------------------------------------

int tf_nms_sets(int32_t n_sets, const int32_t* offsets, const double* boxes, const double* scores,
                const double* thresholds, uint8_t* keep, int32_t* status, void* cuda_stream) {
  // offsets: HOST [n_sets + 1]; payloads device.
  if (n_sets < 0 || (n_sets > 0 && !offsets)) return TF_ARGUMENT;
  if (n_sets == 0) return TF_OK;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  int cap = 1;
  for (int i = 0; i < n_sets; ++i) cap = std::max(cap, offsets[i + 1] - offsets[i]);
  if (cap > 1024) return TF_CAPACITY;
  int* d_off = nullptr;
  if (cudaMallocAsync(&d_off, sizeof(int) * (n_sets + 1), st) != cudaSuccess) return TF_CUDA;
  cudaMemcpyAsync(d_off, offsets, sizeof(int) * (n_sets + 1), cudaMemcpyHostToDevice, st);
  cudaError_t e = launch_nms_sets(n_sets, d_off, boxes, scores, thresholds, keep, status, cap, st);
  cudaFreeAsync(d_off, st);
  return e == cudaSuccess ? TF_OK : TF_CUDA;
}

int tf_lap_dense(int32_t n, const int32_t* shapes, const int64_t* cost_offsets, const double* costs,
                 const int64_t* row_offsets, int32_t* col_for_row, int32_t* status, void* cuda_stream) {
  // shapes / cost_offsets / row_offsets: HOST; costs, col_for_row, status: device.
  if (n < 0 || (n > 0 && (!shapes || !cost_offsets || !row_offsets))) return TF_ARGUMENT;
  if (n == 0) return TF_OK;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  int cap_n = 1;
  long long stride = 1;
  for (int i = 0; i < n; ++i) {
    cap_n = std::max(cap_n, std::max(shapes[2 * i], shapes[2 * i + 1]));
    stride = std::max(stride, static_cast<long long>(shapes[2 * i]) * shapes[2 * i + 1]);
  }
  if (cap_n > 2048) return TF_CAPACITY;
  int* d_shapes = nullptr;
  long long *d_coff = nullptr, *d_roff = nullptr;
  int16_t* pcol = nullptr;
  double* pval = nullptr;
  int* prow = nullptr;
  bool ok = cudaMallocAsync(&d_shapes, sizeof(int) * 2 * n, st) == cudaSuccess &&
            cudaMallocAsync(&d_coff, sizeof(long long) * n, st) == cudaSuccess &&
            cudaMallocAsync(&d_roff, sizeof(long long) * n, st) == cudaSuccess &&
            cudaMallocAsync(&pcol, sizeof(int16_t) * stride * n, st) == cudaSuccess &&
            cudaMallocAsync(&pval, sizeof(double) * stride * n, st) == cudaSuccess &&
            cudaMallocAsync(&prow, sizeof(int) * (cap_n + 1) * static_cast<size_t>(n), st) == cudaSuccess;
  if (!ok) return TF_CUDA;
  cudaMemcpyAsync(d_shapes, shapes, sizeof(int) * 2 * n, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_coff, cost_offsets, sizeof(long long) * n, cudaMemcpyHostToDevice, st);
  cudaMemcpyAsync(d_roff, row_offsets, sizeof(long long) * n, cudaMemcpyHostToDevice, st);
  cudaError_t e = launch_lap_dense(n, d_shapes, d_coff, costs, d_roff, col_for_row, status, cap_n, pcol, pval,
                                   prow, stride, st);
  cudaFreeAsync(d_shapes, st);
  cudaFreeAsync(d_coff, st);
  cudaFreeAsync(d_roff, st);
  cudaFreeAsync(pcol, st);
  cudaFreeAsync(pval, st);
  cudaFreeAsync(prow, st);
  return e == cudaSuccess ? TF_OK : TF_CUDA;
}

int tf_kalman(int32_t op, int32_t n, const tf_config* config, const double* mean_in, const double* cov_in,
              const double* z, double* mean_out, double* cov_out, int32_t* status, void* cuda_stream) {
  if (!config || op < 0 || op > 3 || n < 0) return TF_ARGUMENT;
  return launch_kalman(op, n, make_params(*config), mean_in, cov_in, z, mean_out, cov_out, status,
                       static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess
             ? TF_OK
             : TF_CUDA;
}

int tf_gating(int32_t n_tracks, const double* means, const double* covs, int32_t n_meas, const double* z,
              int32_t metric, const tf_config* config, double* out, int32_t* status, void* cuda_stream) {
  if (!config || n_tracks < 0 || n_meas < 0) return TF_ARGUMENT;
  return launch_gating(n_tracks, means, covs, n_meas, z, metric, make_params(*config), out, status,
                       static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess
             ? TF_OK
             : TF_CUDA;
}

int tf_cosine_cost(int32_t nt, int32_t nd, int32_t dim, const float* te, const float* de, double* out,
                   void* cuda_stream) {
  if (nt < 0 || nd < 0 || dim < 1) return TF_ARGUMENT;
  return launch_cosine_cost(nt, nd, dim, te, de, out, static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess
             ? TF_OK
             : TF_CUDA;
}

int tf_normalize_rows(int32_t n, int32_t dim, const double* in64, const float* in32, int64_t row_stride,
                      int32_t quantize, float* out, int32_t* status, void* cuda_stream) {
  if (n < 0 || dim < 1 || (!in64 && !in32 && n > 0)) return TF_ARGUMENT;
  return launch_normalize_rows(n, dim, in64, in32, row_stride, quantize, out, status,
                               static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess
             ? TF_OK
             : TF_CUDA;
}

int tf_quantize_binary16(int64_t n, const float* in, float* out, int32_t* status, void* cuda_stream) {
  if (n < 0) return TF_ARGUMENT;
  return launch_binary16(n, in, out, status, static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess ? TF_OK
                                                                                                     : TF_CUDA;
}

int tf_smooth_embedding(int32_t n, int32_t dim, const float* old_emb, const float* new_emb, double alpha,
                        float* out, int32_t* status, void* cuda_stream) {
  if (n < 0 || dim < 1) return TF_ARGUMENT;
  return launch_smooth(n, dim, old_emb, new_emb, alpha, 1.0 - alpha, out, status,
                       static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess
             ? TF_OK
             : TF_CUDA;
}

int tf_iou_pairs(int32_t n, const double* a, const double* b, double* out, void* cuda_stream) {
  if (n < 0) return TF_ARGUMENT;
  return launch_iou(n, a, b, out, static_cast<cudaStream_t>(cuda_stream)) == cudaSuccess ? TF_OK : TF_CUDA;
}

}  // extern "C"
