// sm_100a kernels of the decode -> NMS -> association path.
//
//  frame_heads_kernel   one CTA per frame: YOLO-head confidence scan with
//                       warp-ballot ordered compaction, candidate box decode,
//                       bitmask NMS, 128-bit embedding gather + fp64 L2-norm.
//                       (K1+K2+K3 of SURVEY.md section 2, fused: the 8 conf
//                       planes are read once, candidates never leave SMEM.)
//  frame_dets_kernel    same NMS / det-buffer tail for already-parsed rows
//                       (the Tracker.step entry point).
//  associate_kernel     one CTA per stream, persistent over the B frames of an
//                       update: Kalman predict -> gate -> sparse fp64 cosine
//                       cost -> exact LAP -> threshold -> Kalman update, EMA,
//                       lifecycle, births, records (K4..K9).
//  stage kernels        batched nms / lap / kalman / gating / cost / normalize /
//                       binary16 / smooth / iou for the reference's module-level
//                       functions.
#include <algorithm>
#include <climits>
#include <cooperative_groups.h>
#include <map>
#include <mutex>

#include "tf_kernels.cuh"

namespace cg = cooperative_groups;

#include <cstdio>
// Debug: extra CTA barriers at the transitions selected by TF_XSYNC_MASK
// (race bisection; compiled out by default).
#ifndef TF_XSYNC_MASK
#define TF_XSYNC_MASK 0
#endif
#define TF_XSYNC(n)                                   \
  do {                                                \
    if ((TF_XSYNC_MASK >> (n)) & 1) __syncthreads();  \
  } while (0)
#ifdef TF_BOUNDS
#define TF_BCHK(cond, ...)                     \
  do {                                         \
    if (!(cond)) printf("TFBOUND " __VA_ARGS__); \
  } while (0)
#else
#define TF_BCHK(cond, ...) \
  do {                     \
  } while (0)
#endif
namespace tfd {

// Host-side launch helpers: the dynamic shared-memory opt-in of a kernel is
// only ever raised, once per size (cudaFuncSetAttribute costs microseconds
// per call, which shows at small batches; every setter of these kernels goes
// through here so the cache stays true), and the SM count is read once.
static std::mutex g_attr_mu;
static std::map<std::pair<const void*, int>, int> g_smem_set;     // (kernel, device) -> bytes set
static void set_smem(const void* fn, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(g_attr_mu);
  const auto key = std::make_pair(fn, dev);
  auto it = g_smem_set.find(key);
  if (it != g_smem_set.end() && it->second >= static_cast<int>(bytes)) return;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) == cudaSuccess)
    g_smem_set[key] = static_cast<int>(bytes);
}
static int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// ============================================================================
// Frame stage (heads)
// ============================================================================

struct ScaleDev {
  const float* head;             // confidence planes (channels 6a+4, 6a+5)
  long long hs_n, hs_c;
  const float* delta;            // box deltas (channels 6a+0..3)
  long long ds_n, ds_c;
  const float* emb;
  long long es_n, es_c, es_h, es_w;
  int H, W, stride, pad;
  float aw[4], ah[4];
};

struct FrameArgs {
  ScaleDev sc[3];
  double scale_inv, pad_x, pad_y;
  int frames;
  int cap_cand, cap_det, words;
  DetBuf det;
  // overlapped mode (ready == nullptr: one CTA per frame)
  unsigned* ready;               // [frames] the update's epoch once frame f is decoded
  unsigned epoch;
  int* ticket;                   // [2] work counter, exit counter (left at 0)
  const int* order;              // the association's block -> stream order (nullptr = identity)
  int first_wave, streams, B;
};

// Shared-memory plan of frame_heads_kernel (bytes computed by frame_smem_bytes()).
struct FramePlan {
  int nchunks;
  size_t off_masks, off_code, off_box, off_score, off_alive, off_sorted, off_nmask, off_keep, off_pos,
      total;
};

__host__ __device__ inline size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

__host__ __device__ inline FramePlan frame_plan(int total_anchors, int cap_cand, int words) {
  FramePlan p;
  // confidence scan groups: 128 anchors of one (scale, anchor) plane each,
  // so at most total/128 + 12 groups; four 32-bit ballots per group
  p.nchunks = (total_anchors + 127) / 128 + 12;
  size_t o = 0;
  p.off_masks = o;  o = align16(o + 16 * static_cast<size_t>(p.nchunks));
  p.off_code = o;   o = align16(o + sizeof(int) * cap_cand);
  p.off_box = o;    o = align16(o + sizeof(double) * 4 * cap_cand);
  p.off_score = o;  o = align16(o + sizeof(double) * cap_cand);
  p.off_alive = o;  o = align16(o + cap_cand);
  p.off_sorted = o; o = align16(o + sizeof(int16_t) * cap_cand);
  p.off_nmask = o;  o = align16(o + sizeof(unsigned long long) * cap_cand * words);
  p.off_keep = o;   o = align16(o + cap_cand);
  p.off_pos = o;    o = align16(o + sizeof(int16_t) * cap_cand);
  p.total = o;
  return p;
}

// Element access of the head / embedding inputs: fp32, or binary16 (the
// MIXED-precision input mode: every fp16 value is exact in fp32 / fp64, so the
// decode and the decisions downstream are those of the same values in fp32).
template <typename T> struct Elt;
template <> struct Elt<float> {
  static constexpr int kVecBytes = 16;                 // 4 elements per vector load
  static __device__ __forceinline__ float ld(const float* p) { return __ldg(p); }
  static __device__ __forceinline__ float ldcs(const float* p) { return __ldcs(p); }
  static __device__ __forceinline__ float4 ld4(const float* p) { return __ldg(reinterpret_cast<const float4*>(p)); }
  static __device__ __forceinline__ float4 ld4cs(const float* p) { return __ldcs(reinterpret_cast<const float4*>(p)); }
};
template <> struct Elt<__half> {
  static constexpr int kVecBytes = 8;
  static __device__ __forceinline__ float ld(const __half* p) {
    return __half2float(__ushort_as_half(__ldg(reinterpret_cast<const unsigned short*>(p))));
  }
  static __device__ __forceinline__ float ldcs(const __half* p) {
    return __half2float(__ushort_as_half(__ldcs(reinterpret_cast<const unsigned short*>(p))));
  }
  static __device__ __forceinline__ float4 cvt(uint2 u) {
    const float2 a = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
    return make_float4(a.x, a.y, b.x, b.y);
  }
  static __device__ __forceinline__ float4 ld4(const __half* p) { return cvt(__ldg(reinterpret_cast<const uint2*>(p))); }
  static __device__ __forceinline__ float4 ld4cs(const __half* p) { return cvt(__ldcs(reinterpret_cast<const uint2*>(p))); }
};

// Gather one embedding row (warp-cooperative), fp64 sum of squares, optional
// binary16 round trip; writes the fp32 unit vector to `out` when non-null.
// Mirrors normalize (tf/core.py:100-111) and _quantize_detection
// (tf/pipeline.py:436-441). Returns a tf_status code (0 ok). The norm of every
// row is checked even when `out` is null (parse_output normalises all rows).
template <typename T>
__device__ int gather_normalize(const T* src, long long stride, int dim, int quantize, float* out) {
  const int lane = lane_id();
  const bool vec = (stride == 1) && ((reinterpret_cast<uintptr_t>(src) & (Elt<T>::kVecBytes - 1)) == 0) && (dim % 4 == 0) &&
                   (out == nullptr || (reinterpret_cast<uintptr_t>(out) & 15) == 0);
  double ss = 0.0;
  bool finite = true;
  if (vec && dim == 512 && !quantize) {
    // the common row: 16 values per lane held in registers, one read
    float4 q[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = Elt<T>::ld4(src + 4 * (lane + 32 * j));
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      finite = finite && isfinite(q[j].x) && isfinite(q[j].y) && isfinite(q[j].z) && isfinite(q[j].w);
      ss = fma(static_cast<double>(q[j].x), static_cast<double>(q[j].x), ss);
      ss = fma(static_cast<double>(q[j].y), static_cast<double>(q[j].y), ss);
      ss = fma(static_cast<double>(q[j].z), static_cast<double>(q[j].z), ss);
      ss = fma(static_cast<double>(q[j].w), static_cast<double>(q[j].w), ss);
    }
    ss = warp_sum(ss);
    finite = __all_sync(FULL, finite);
    if (!finite) return TF_DEGENERATE_EMBEDDING;
    const double norm = sqrt(ss);
    if (norm < 1e-12) return TF_DEGENERATE_EMBEDDING;
    if (out == nullptr) return TF_OK;
    float4* o4 = reinterpret_cast<float4*>(out);
    const double rn = __drcp_rn(norm);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float4 r;
      r.x = static_cast<float>(div_by(static_cast<double>(q[j].x), norm, rn));
      r.y = static_cast<float>(div_by(static_cast<double>(q[j].y), norm, rn));
      r.z = static_cast<float>(div_by(static_cast<double>(q[j].z), norm, rn));
      r.w = static_cast<float>(div_by(static_cast<double>(q[j].w), norm, rn));
      o4[lane + 32 * j] = r;
    }
    return TF_OK;
  }
  if (vec) {
    for (int i = lane; i < dim / 4; i += 32) {
      float4 q = Elt<T>::ld4(src + 4 * i);
      double a = q.x, b = q.y, c = q.z, d = q.w;
      finite = finite && isfinite(q.x) && isfinite(q.y) && isfinite(q.z) && isfinite(q.w);
      ss = fma(a, a, ss);
      ss = fma(b, b, ss);
      ss = fma(c, c, ss);
      ss = fma(d, d, ss);
    }
  } else {
    for (int i = lane; i < dim; i += 32) {
      float x = Elt<T>::ld(src + static_cast<long long>(i) * stride);
      finite = finite && isfinite(x);
      double a = x;
      ss = fma(a, a, ss);
    }
  }
  ss = warp_sum(ss);
  finite = __all_sync(FULL, finite);
  if (!finite) return TF_DEGENERATE_EMBEDDING;
  const double norm = sqrt(ss);
  if (norm < 1e-12) return TF_DEGENERATE_EMBEDDING;
  if (!quantize) {
    if (out == nullptr) return TF_OK;
    if (vec) {
      float4* o4 = reinterpret_cast<float4*>(out);
      const double rn = __drcp_rn(norm);
      for (int i = lane; i < dim / 4; i += 32) {
        float4 q = Elt<T>::ld4(src + 4 * i);
        float4 r;
        r.x = static_cast<float>(div_by(static_cast<double>(q.x), norm, rn));
        r.y = static_cast<float>(div_by(static_cast<double>(q.y), norm, rn));
        r.z = static_cast<float>(div_by(static_cast<double>(q.z), norm, rn));
        r.w = static_cast<float>(div_by(static_cast<double>(q.w), norm, rn));
        o4[i] = r;
      }
    } else {
      for (int i = lane; i < dim; i += 32)
        out[i] = static_cast<float>(static_cast<double>(Elt<T>::ld(src + static_cast<long long>(i) * stride)) / norm);
    }
    return TF_OK;
  }
  // MIXED: fp32 unit vector -> binary16 (RNE) -> fp32 -> normalize again.
  double ss2 = 0.0;
  bool inrange = true;
  for (int i = lane; i < dim; i += 32) {
    float u = static_cast<float>(static_cast<double>(Elt<T>::ld(src + static_cast<long long>(i) * stride)) / norm);
    inrange = inrange && fabsf(u) <= 65504.0f;
    double h = __half2float(__float2half_rn(u));
    ss2 += h * h;
  }
  ss2 = warp_sum(ss2);
  if (!__all_sync(FULL, inrange)) return TF_PRECISION_OVERFLOW;
  const double n2 = sqrt(ss2);
  if (n2 < 1e-12) return TF_DEGENERATE_EMBEDDING;
  if (out == nullptr) return TF_OK;
  for (int i = lane; i < dim; i += 32) {
    float u = static_cast<float>(static_cast<double>(Elt<T>::ld(src + static_cast<long long>(i) * stride)) / norm);
    double h = __half2float(__float2half_rn(u));
    out[i] = static_cast<float>(h / n2);
  }
  return TF_OK;
}

// Block size is a template parameter: 1024 threads when there are few frames
// (each CTA's own latency matters), 256 when frames outnumber the SMs (more
// CTAs per SM overlap one another's scan / NMS / gather phases): B200, cfg1
// 32 frames 46 -> 39 us, cfg4 4,096 frames 0.71 -> 0.63 ms.
#ifndef TF_FRAME_MINB
#define TF_FRAME_MINB 4   // 256-thread CTAs: <= 64 registers, 4 CTAs per SM (cfg4: 5 -> 0.58 ms with spills, 1 -> 90 registers, 0.88 ms)
#endif
#ifdef TF_FRAME_TIMERS
// diagnostics: clock64 at the phase boundaries of frame 0's leader CTA, printed per launch
#define TF_FT(i) if (f == 0 && crank == 0 && threadIdx.x == 0) ft[i] = clock64();
#else
#define TF_FT(i)
#endif
// One frame: scan, decode, NMS, gather (the body of frame_heads_kernel).
template <typename T, int kThreads>
__device__ __forceinline__ void frame_heads_body(const FrameArgs& a, const Params& P, const int f, cg::cluster_group cl,
                                                 const int CR, const int crank) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, lane = lane_id(), wid = warp_id(), nw = n_warps();
#ifdef TF_FRAME_TIMERS
  long long ft[10] = {0};
#endif
  TF_FT(0);

  __shared__ const T* s_bg[12];
  __shared__ const T* s_fg[12];
  __shared__ int s_start[13];
  __shared__ int s_gstart[13];           // first scan group of each plane
  __shared__ int s_vec[12];              // plane pair is 16-byte aligned (float4 loads)
  __shared__ int s_warp[33];
  __shared__ int s_misc[4];

  if (tid < 12) {
    int si = tid / 4, an = tid % 4;
    const ScaleDev& sc = a.sc[si];
    const T* base = reinterpret_cast<const T*>(sc.head) + static_cast<long long>(f) * sc.hs_n;
    s_bg[tid] = base + static_cast<long long>(6 * an + 4) * sc.hs_c;
    s_fg[tid] = base + static_cast<long long>(6 * an + 5) * sc.hs_c;
  }
  if (tid == 0) {
    int acc = 0;
    for (int si = 0; si < 3; ++si)
      for (int an = 0; an < 4; ++an) {
        s_start[si * 4 + an] = acc;
        acc += a.sc[si].H * a.sc[si].W;
      }
    s_start[12] = acc;
    int gacc = 0;
    for (int p = 0; p < 12; ++p) {
      s_gstart[p] = gacc;
      gacc += (s_start[p + 1] - s_start[p] + 127) / 128;
    }
    s_gstart[12] = gacc;
    s_misc[0] = STATUS_CLEAR;
  }
  __syncthreads();
  if (tid < 12) {
    const int hw = s_start[tid + 1] - s_start[tid];
    s_vec[tid] = ((reinterpret_cast<uintptr_t>(s_bg[tid]) | reinterpret_cast<uintptr_t>(s_fg[tid])) &
                  (Elt<T>::kVecBytes - 1)) == 0 &&
                 (hw & 3) == 0;
  }
  __syncthreads();
  const int total = s_start[12];
  const FramePlan plan = frame_plan(total, a.cap_cand, a.words);
  int* ccode = reinterpret_cast<int*>(smem + plan.off_code);
  double* cbox = reinterpret_cast<double*>(smem + plan.off_box);
  double* cscore = reinterpret_cast<double*>(smem + plan.off_score);
  uint8_t* calive = smem + plan.off_alive;
  int16_t* csorted = reinterpret_cast<int16_t*>(smem + plan.off_sorted);
  unsigned long long* nmask = reinterpret_cast<unsigned long long*>(smem + plan.off_nmask);
  uint8_t* ckeep = smem + plan.off_keep;
  int16_t* cpos = reinterpret_cast<int16_t*>(smem + plan.off_pos);

  TF_FT(1);
  // ---- pass 1: confidence scan ---------------------------------------------
  // The 12 (scale, anchor) background / foreground plane pairs are split into
  // groups of 128 anchors; a lane owns 4 consecutive anchors (one float4 of
  // each plane when the planes are 16-byte aligned) and a warp keeps TF_SCAN_U
  // groups of loads in flight. Each group stores four ballots (bit l of
  // ballot i = anchor 4l + i) so pass 2 ranks candidates without re-reading.
  const uint4* gmask_ro = reinterpret_cast<const uint4*>(smem + plan.off_masks);
  uint4* gmasks = reinterpret_cast<uint4*>(smem + plan.off_masks);
  const int NG = s_gstart[12];
  const int nwc = nw * CR, gw = crank * nw + wid;            // the cluster's warps share the groups
  const int per_warp = (NG + nwc - 1) / nwc;
  const int g0 = min(NG, gw * per_warp), g1 = min(NG, g0 + per_warp);
  uint4* out_masks = CR > 1 ? cl.map_shared_rank(gmasks, 0) : gmasks;
  const double lim = P.conf_logit;
  const bool lim_zero = lim == 0.0;
  int count = 0;
  constexpr int U = 4;
  {
    int pl = 0;
    for (int g = g0; g < g1; g += U) {
      float4 bgv[U], fgv[U];
#pragma unroll
      for (int k = 0; k < U; ++k) {
        const int gg = g + k;
        bgv[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        fgv[k] = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        if (gg < g1) {
          while (gg >= s_gstart[pl + 1]) ++pl;
          const int hw = s_start[pl + 1] - s_start[pl];
          const int pos = (gg - s_gstart[pl]) * 128 + 4 * lane;
          if (s_vec[pl]) {
            if (pos < hw) {
              bgv[k] = Elt<T>::ld4cs(s_bg[pl] + pos);
              fgv[k] = Elt<T>::ld4cs(s_fg[pl] + pos);
            }
          } else {
            const T* pb = s_bg[pl] + pos;
            const T* pf = s_fg[pl] + pos;
            if (pos < hw) { bgv[k].x = Elt<T>::ldcs(pb); fgv[k].x = Elt<T>::ldcs(pf); }
            if (pos + 1 < hw) { bgv[k].y = Elt<T>::ldcs(pb + 1); fgv[k].y = Elt<T>::ldcs(pf + 1); }
            if (pos + 2 < hw) { bgv[k].z = Elt<T>::ldcs(pb + 2); fgv[k].z = Elt<T>::ldcs(pf + 2); }
            if (pos + 3 < hw) { bgv[k].w = Elt<T>::ldcs(pb + 3); fgv[k].w = Elt<T>::ldcs(pf + 3); }
          }
        }
      }
#pragma unroll
      for (int k = 0; k < U; ++k) {
        if (g + k >= g1) break;
        unsigned m0, m1, m2, m3;
        if (lim_zero) {
          // logit(0.5) = 0: the sign of an fp32 difference is the sign of
          // the exact one (gradual underflow; inf - inf is NaN either way),
          // so this equals the fp64 test without the fp32 -> fp64 conversions
          m0 = __ballot_sync(FULL, fgv[k].x - bgv[k].x >= 0.0f);
          m1 = __ballot_sync(FULL, fgv[k].y - bgv[k].y >= 0.0f);
          m2 = __ballot_sync(FULL, fgv[k].z - bgv[k].z >= 0.0f);
          m3 = __ballot_sync(FULL, fgv[k].w - bgv[k].w >= 0.0f);
        } else {
          m0 = __ballot_sync(FULL, (static_cast<double>(fgv[k].x) - static_cast<double>(bgv[k].x)) >= lim);
          m1 = __ballot_sync(FULL, (static_cast<double>(fgv[k].y) - static_cast<double>(bgv[k].y)) >= lim);
          m2 = __ballot_sync(FULL, (static_cast<double>(fgv[k].z) - static_cast<double>(bgv[k].z)) >= lim);
          m3 = __ballot_sync(FULL, (static_cast<double>(fgv[k].w) - static_cast<double>(bgv[k].w)) >= lim);
        }
        if (lane == 0) out_masks[g + k] = make_uint4(m0, m1, m2, m3);
        count += __popc(m0) + __popc(m1) + __popc(m2) + __popc(m3);
      }
    }
  }
  TF_FT(2);
  // pass-2 ranges are the leader's own warps' over all groups
  int p0 = g0, p1 = g1;
  if (CR > 1) {
    cl.sync();                                     // every CTA's ballots are in the leader
    if (crank != 0) return;
    const int pw = (NG + nw - 1) / nw;
    p0 = min(NG, wid * pw);
    p1 = min(NG, p0 + pw);
    count = 0;
    for (int gg = p0 + lane; gg < p1; gg += 32) {
      const uint4 m = gmask_ro[gg];
      count += __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
    }
    count = __reduce_add_sync(FULL, static_cast<unsigned>(count));
  }
  if (lane == 0) s_warp[wid] = count;
  __syncthreads();
  if (wid == 0) {
    int v = lane < nw ? s_warp[lane] : 0, incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane < nw) s_warp[lane] = incl - v;
    if (lane == 31) s_warp[32] = incl;
  }
  __syncthreads();
  const int C_all = s_warp[32];
  const int C = min(C_all, a.cap_cand);
  if (tid == 0 && C_all > a.cap_cand) flag_error(&s_misc[0], 0, TF_CAPACITY);

  TF_FT(3);
  // ---- pass 2: ordered compaction of candidate codes (anchor order) --------
  {
    int base = s_warp[wid];
    int pl = 0;
    const unsigned lt = (1u << lane) - 1u;
    for (int gg = p0; gg < p1; ++gg) {
      const uint4 m = gmask_ro[gg];
      const int tot = __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
      if (tot == 0) continue;
      while (gg >= s_gstart[pl + 1]) ++pl;
      int r = base + __popc(m.x & lt) + __popc(m.y & lt) + __popc(m.z & lt) + __popc(m.w & lt);
      const int a0 = s_start[pl] + (gg - s_gstart[pl]) * 128 + 4 * lane;
      if ((m.x >> lane) & 1u) { if (r < C) ccode[r] = a0; ++r; }
      if ((m.y >> lane) & 1u) { if (r < C) ccode[r] = a0 + 1; ++r; }
      if ((m.z >> lane) & 1u) { if (r < C) ccode[r] = a0 + 2; ++r; }
      if ((m.w >> lane) & 1u) { if (r < C) ccode[r] = a0 + 3; ++r; }
      base += tot;
    }
  }
  __syncthreads();

  TF_FT(4);
  // ---- candidate decode (sigmoid/exp boxes, letterbox inverse) -------------
  for (int r = tid; r < C; r += blockDim.x) {
    int g = ccode[r];
    int p = 0;
    while (g >= s_start[p + 1]) ++p;
    const int si = p >> 2, an = p & 3;
    const ScaleDev& sc = a.sc[si];
    const int pos = g - s_start[p];
    const int y = pos / sc.W, x = pos - y * sc.W;
    const T* base = reinterpret_cast<const T*>(sc.head) + static_cast<long long>(f) * sc.hs_n + pos;
    const T* dbase = reinterpret_cast<const T*>(sc.delta) + static_cast<long long>(f) * sc.ds_n + pos;
    const double tx = Elt<T>::ld(dbase + (6 * an + 0) * sc.ds_c);
    const double ty = Elt<T>::ld(dbase + (6 * an + 1) * sc.ds_c);
    const double tw = Elt<T>::ld(dbase + (6 * an + 2) * sc.ds_c);
    const double th = Elt<T>::ld(dbase + (6 * an + 3) * sc.ds_c);
    const double xl = static_cast<double>(Elt<T>::ld(base + (6 * an + 5) * sc.hs_c)) -
                      static_cast<double>(Elt<T>::ld(base + (6 * an + 4) * sc.hs_c));
    double cx = (static_cast<double>(x) + 1.0 / (1.0 + exp(-tx))) * static_cast<double>(sc.stride);
    double cy = (static_cast<double>(y) + 1.0 / (1.0 + exp(-ty))) * static_cast<double>(sc.stride);
    double bw = static_cast<double>(sc.aw[an]) * exp(tw);
    double bh = static_cast<double>(sc.ah[an]) * exp(th);
    cx = (cx - a.pad_x) * a.scale_inv;
    cy = (cy - a.pad_y) * a.scale_inv;
    bw = bw * a.scale_inv;
    bh = bh * a.scale_inv;
    double bx = cx - bw / 2.0, by = cy - bh / 2.0;
    cbox[4 * r + 0] = bx;
    cbox[4 * r + 1] = by;
    cbox[4 * r + 2] = bw;
    cbox[4 * r + 3] = bh;
    const double score = 1.0 / (1.0 + exp(-xl));
    cscore[r] = score;
    calive[r] = score >= P.conf_threshold;
    if (!(isfinite(bx) && isfinite(by) && isfinite(bw) && isfinite(bh)) || !(bw > 0.0) || !(bh > 0.0))
      flag_error(&s_misc[0], r + 1, TF_INVALID_BOX);
  }
  __syncthreads();

  TF_FT(5);
  // ---- NMS ------------------------------------------------------------------
  block_nms(C, cbox, cscore, calive, P.nms_iou, csorted, nmask, a.words, ckeep, &s_misc[1]);
  TF_FT(6);
  const int K_all = block_rank(C, [&](int i) { return ckeep[i] != 0; }, cpos, s_warp);
  const int K = min(K_all, a.cap_det);
  if (tid == 0 && K_all > a.cap_det) flag_error(&s_misc[0], 0, TF_CAPACITY);

  // ---- det buffer: measurement, objectness, code; embeddings -------------
  const long long fbase = static_cast<long long>(f) * a.cap_det;
  for (int r = tid; r < C; r += blockDim.x) {
    int k = cpos[r];
    if (k < 0 || k >= K) continue;
    double m[4];
    box_to_meas(&cbox[4 * r], m);
    double* dm = a.det.meas + (fbase + k) * 4;
    dm[0] = m[0]; dm[1] = m[1]; dm[2] = m[2]; dm[3] = m[3];
    a.det.obj[fbase + k] = cscore[r];
    a.det.code[fbase + k] = ccode[r];
  }
  // parse_output normalises every row (tf/postproc.py:31-33), so every
  // candidate's norm is checked; only kept ones are written.
  const int D = P.dim;
  for (int r = wid; r < C; r += nw) {
    int g = ccode[r];
    int p = 0;
    while (g >= s_start[p + 1]) ++p;
    const ScaleDev& sc = a.sc[p >> 2];
    const int pos = g - s_start[p];
    const int y = pos / sc.W, x = pos - y * sc.W;
    const T* src = reinterpret_cast<const T*>(sc.emb) + static_cast<long long>(f) * sc.es_n + static_cast<long long>(y) * sc.es_h +
                       static_cast<long long>(x) * sc.es_w;
    int k = cpos[r];
    float* out = (k >= 0 && k < K) ? a.det.emb + (fbase + k) * D : nullptr;
    int st = gather_normalize(src, sc.es_c, D, P.quantize, out);
    if (st != TF_OK && lane == 0) flag_error(&s_misc[0], r + 1, st);
  }
  TF_FT(7);
  __syncthreads();
  TF_FT(8);
#ifdef TF_FRAME_TIMERS
  if (f == 0 && crank == 0 && tid == 0)
    printf("TFFT C=%d K=%d setup %lld scan %lld sync %lld rank %lld decode %lld nms %lld gather %lld tail %lld\n", C, K,
           ft[1] - ft[0], ft[2] - ft[1], ft[3] - ft[2], ft[4] - ft[3], ft[5] - ft[4], ft[6] - ft[5], ft[7] - ft[6],
           ft[8] - ft[7]);
#endif
  if (tid == 0) {
    a.det.count[f] = K;
    a.det.cand_count[f] = C_all;
    int st = s_misc[0];
    a.det.status[f] = (st == STATUS_CLEAR) ? 0 : (st & 0xff);
  }
}

// Frame of the i-th visit in overlapped mode: the association's block order
// (a.order: longest-first when it is used, else identity) in chunks of
// first_wave blocks, frame-major inside a chunk, so the streams whose CTAs
// start first get their frames 0, 1, ... first and each association CTA
// finds its next frame decoded before it needs it.
__device__ __forceinline__ int visit_frame(const FrameArgs& a, int i) {
  const int W = a.first_wave, B = a.B;
  const int chunk = i / (W * B), within = i - chunk * W * B;
  const int nc = min(W, a.streams - chunk * W);
  const int b = within / nc;
  const int p = chunk * W + (within - b * nc);
  const int ls = a.order ? a.order[p] : p;
  return ls * B + b;
}

__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// With few frames a thread-block cluster scans each frame: every CTA takes a
// share of the anchor groups and stores its ballots into the leader CTA's
// shared memory (DSMEM); the leader then ranks, decodes, suppresses and
// gathers alone. One CTA per frame (cluster size 1) otherwise.
//
// Overlapped mode (a.ready != nullptr; many frames, no cluster): a persistent
// grid takes frames from a work counter in visit_frame order and publishes
// each finished frame with a release store of the update's epoch into
// a.ready[f]. The association grid (next on the stream, programmatic
// dependent launch) starts at once and waits per frame on these flags instead
// of on this grid's completion, so decode and association overlap within one
// update. No deadlock: the association is launched only once every CTA of
// this grid is resident (all of them trigger at entry), and this grid never
// waits on it.
template <typename T, int kThreads>
__global__ void __launch_bounds__(kThreads, kThreads == 256 ? TF_FRAME_MINB : 1) frame_heads_kernel(FrameArgs a, Params P) {
  cg::cluster_group cl = cg::this_cluster();
  const int CR = static_cast<int>(cl.num_blocks());
  const int crank = static_cast<int>(cl.block_rank());
  if (a.ready == nullptr) {
    frame_heads_body<T, kThreads>(a, P, blockIdx.x / CR, cl, CR, crank);
    return;
  }
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  __shared__ int s_visit;
  for (;;) {
    if (threadIdx.x == 0) s_visit = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int i = s_visit;
    if (i >= a.frames) break;
    const int f = visit_frame(a, i);
    frame_heads_body<T, kThreads>(a, P, f, cl, 1, 0);
    __syncthreads();                          // every thread's outputs of frame f are written
    if (threadIdx.x == 0) {
      __threadfence();
      st_release_gpu(a.ready + f, a.epoch);
    }
  }
  if (threadIdx.x == 0 && atomicAdd(a.ticket + 1, 1) == static_cast<int>(gridDim.x) - 1) {
    a.ticket[0] = 0;                          // the last CTA out resets the counters
    a.ticket[1] = 0;
  }
}

// ============================================================================
// Frame stage (already-parsed detections, the Tracker.step entry)
// ============================================================================
struct RowsArgs {
  const double* boxes;
  const double* obj;
  const float* emb;
  const uint8_t* has_emb;          // null: every row has an embedding
  const int* offsets;              // [frames + 1] row ranges (batched entry), or null: one frame of n rows
  int n, cap_cand, cap_det, words;
  int normalize;                   // 1: rows are raw parse_output input (normalise, tf/postproc.py:31-33)
  DetBuf det;
};

// One CTA per frame: filter_confidence + NMS + detection buffer for rows that
// are already decoded (Tracker.step, or the batched detection-file source).
__global__ void __launch_bounds__(512) frame_dets_kernel(RowsArgs a, Params P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int tid = threadIdx.x, wid = warp_id(), nw = n_warps(), lane = lane_id();
  __shared__ int s_warp[33];
  __shared__ int s_misc[4];
  const int f = blockIdx.x;
  const int r0 = a.offsets ? a.offsets[f] : 0;
  const int C_all = a.offsets ? a.offsets[f + 1] - r0 : a.n;
  const int C = min(C_all, a.cap_cand);
  const double* boxes = a.boxes + 4LL * r0;
  const double* obj = a.obj + r0;
  const uint8_t* has = a.has_emb ? a.has_emb + r0 : nullptr;
  const int D = P.dim;
  const float* emb = a.emb + static_cast<long long>(r0) * D;
  const long long fb = static_cast<long long>(f) * a.cap_det;
  const FramePlan plan = frame_plan(0, a.cap_cand, a.words);
  double* cbox = reinterpret_cast<double*>(smem + plan.off_box);
  double* cscore = reinterpret_cast<double*>(smem + plan.off_score);
  uint8_t* calive = smem + plan.off_alive;
  int16_t* csorted = reinterpret_cast<int16_t*>(smem + plan.off_sorted);
  unsigned long long* nmask = reinterpret_cast<unsigned long long*>(smem + plan.off_nmask);
  uint8_t* ckeep = smem + plan.off_keep;
  int16_t* cpos = reinterpret_cast<int16_t*>(smem + plan.off_pos);
  if (tid == 0) {
    s_misc[0] = STATUS_CLEAR;
    if (C_all > a.cap_cand) flag_error(&s_misc[0], 0, TF_CAPACITY);
  }
  for (int r = tid; r < C; r += blockDim.x) {
    for (int q = 0; q < 4; ++q) cbox[4 * r + q] = boxes[4 * r + q];
    cscore[r] = obj[r];
    calive[r] = obj[r] >= P.conf_threshold;
  }
  __syncthreads();
  block_nms(C, cbox, cscore, calive, P.nms_iou, csorted, nmask, a.words, ckeep, &s_misc[1]);
  const int K_all = block_rank(C, [&](int i) { return ckeep[i] != 0; }, cpos, s_warp);
  const int K = min(K_all, a.cap_det);
  if (tid == 0 && K_all > a.cap_det) flag_error(&s_misc[0], 0, TF_CAPACITY);
  for (int r = tid; r < C; r += blockDim.x) {
    int k = cpos[r];
    if (k < 0 || k >= K) continue;
    if (has && !has[r]) flag_error(&s_misc[0], r + 1, TF_DIMENSION);
    double m[4];
    box_to_meas(&cbox[4 * r], m);
    double* dm = a.det.meas + (fb + k) * 4;
    dm[0] = m[0]; dm[1] = m[1]; dm[2] = m[2]; dm[3] = m[3];
    a.det.obj[fb + k] = cscore[r];
    a.det.code[fb + k] = r;
  }
  for (int r = wid; r < C; r += nw) {
    int k = cpos[r];
    const bool kept = k >= 0 && k < K;
    if (a.normalize) {
      // parse_output normalises every row (and raises on any degenerate one)
      const int stn = gather_normalize<float>(emb + static_cast<long long>(r) * D, 1, D, P.quantize,
                                              kept ? a.det.emb + (fb + k) * D : nullptr);
      if (stn != TF_OK && lane == 0) flag_error(&s_misc[0], r + 1, stn);
      continue;
    }
    if (!kept || (has && !has[r])) continue;
    const float* src = emb + static_cast<long long>(r) * D;
    float* dst = a.det.emb + (fb + k) * D;
    for (int i = lane; i < D; i += 32) dst[i] = src[i];
  }
  __syncthreads();
  if (tid == 0) {
    a.det.count[f] = K;
    a.det.cand_count[f] = C_all;
    int st = s_misc[0];
    a.det.status[f] = (st == STATUS_CLEAR) ? 0 : (st & 0xff);
  }
}

// ============================================================================
// Association: one persistent CTA per stream over the B frames of an update.
// ============================================================================

constexpr int kFrameTable = 64;   // frames per update whose scalars are staged in shared memory

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

struct AssocPlan {
  size_t off_id, off_lost, off_last, off_mean, off_cov, off_mcost, off_state, off_hits,
      off_slot, off_mdet, off_rowptr, off_flag, off_npos, off_rpos, off_dm, off_dobj, off_dm2, off_dobj2, off_drow, off_dpos, off_gmask,
      off_ecol, off_erow, off_eval, off_u, off_v, off_dist, off_crow, off_path, off_r4c, off_c4r, off_rem,
      off_vr, off_vc, off_lab, off_cnr, off_cnc, off_cne, off_croot, off_coff, off_cpos, off_crows, off_ccols,
      off_cmap, off_rcol, off_rmap, off_lrp, off_eoff, off_il, off_epos, off_elist, off_pcmin, off_prmin, off_pccnt, off_pcdeg, off_pcrow, off_prdeg, off_prcnt, off_prc1,
      off_pra, off_pca, off_pkr, off_pkc, off_emas, off_fstk, total;
};

__host__ __device__ inline AssocPlan assoc_plan(int T, int K, int E) {
  AssocPlan p;
  const int NN = T + K;
  const int KW = (K + 31) / 32;
  size_t o = 0;
#define TF_TAKE(field, bytes) p.field = o; o = align16(o + (bytes));
  TF_TAKE(off_id, 8 * T)
  TF_TAKE(off_lost, 8 * T)
  TF_TAKE(off_last, 8 * T)
  TF_TAKE(off_mean, 8 * 8 * T)
  TF_TAKE(off_cov, 8 * 12 * T)
  TF_TAKE(off_mcost, 8 * T)
  TF_TAKE(off_state, 4 * T)
  TF_TAKE(off_hits, 4 * T)
  TF_TAKE(off_slot, 4 * T)
  TF_TAKE(off_mdet, 4 * T)
  TF_TAKE(off_rowptr, 4 * (T + 1))
  TF_TAKE(off_flag, 4 * T)
  TF_TAKE(off_npos, 2 * (T > K ? T : K))
  TF_TAKE(off_rpos, 2 * T)
  TF_TAKE(off_dm, 8 * 4 * K)
  TF_TAKE(off_dobj, 8 * K)
  TF_TAKE(off_dm2, 8 * 4 * K)     // second buffer: frame b + 1 is prefetched while frame b runs
  TF_TAKE(off_dobj2, 8 * K)
  TF_TAKE(off_drow, 4 * K)
  TF_TAKE(off_dpos, 2 * K)
  TF_TAKE(off_emas, 4 * K)        // EMA work list of the frame (det -> pool slot), read by followers
  TF_TAKE(off_fstk, 4 * T)        // free embedding-slot stack of the stream (kept on chip for the launch)
  TF_TAKE(off_ecol, 2 * E)
  TF_TAKE(off_erow, 2 * E)
  TF_TAKE(off_eval, 8 * E)
  // LAP scratch: N for the full solve, or disjoint per-component slices (sum <= T + K)
  TF_TAKE(off_u, 8 * NN)
  TF_TAKE(off_v, 8 * NN)
  TF_TAKE(off_dist, 8 * NN)
  TF_TAKE(off_crow, 8 * NN)
  TF_TAKE(off_path, 2 * NN)
  TF_TAKE(off_r4c, 2 * NN)
  TF_TAKE(off_c4r, 2 * NN)
  TF_TAKE(off_rem, 2 * NN)
  TF_TAKE(off_vr, 2 * (2 * NN + 1))
  TF_TAKE(off_vc, 2 * (2 * NN + 1))
  // peeling kill flags persist (zero) across frames: outside the shared region
  TF_TAKE(off_pkr, T)
  TF_TAKE(off_pkc, K)
  // connected components / peeling; the gate bitmask and the gate factors
  // (dead once the CSR is built) share this region
  const size_t ustart = o;
  p.off_gmask = ustart;
  p.off_il = align16(ustart + 4 * T * KW);
  TF_TAKE(off_lab, 4 * NN)
  TF_TAKE(off_cnr, 4 * NN)
  TF_TAKE(off_cnc, 4 * NN)
  TF_TAKE(off_cne, 4 * NN)
  TF_TAKE(off_croot, 4 * NN)
  TF_TAKE(off_coff, 4 * (NN + 1))
  TF_TAKE(off_cpos, 2 * NN)
  TF_TAKE(off_crows, 2 * NN)
  TF_TAKE(off_ccols, 2 * NN)
  TF_TAKE(off_cmap, 2 * K)
  TF_TAKE(off_rcol, 2 * T)
  TF_TAKE(off_rmap, 2 * T)
  TF_TAKE(off_lrp, 4 * (2 * NN + 1))
  TF_TAKE(off_eoff, 4 * (NN + 1))
  TF_TAKE(off_epos, 2 * E)
  TF_TAKE(off_elist, 2 * E)
  // forced-pair peeling
  TF_TAKE(off_pcmin, 8 * K)
  TF_TAKE(off_prmin, 8 * T)
  TF_TAKE(off_pccnt, 4 * K)
  TF_TAKE(off_pcdeg, 4 * K)
  TF_TAKE(off_pcrow, 4 * K)
  TF_TAKE(off_prdeg, 4 * T)
  TF_TAKE(off_prcnt, 4 * T)
  TF_TAKE(off_prc1, 4 * T)
  TF_TAKE(off_pra, T)
  TF_TAKE(off_pca, K)
  if (o < align16(p.off_il + 32 * T)) o = align16(p.off_il + 32 * T);
#undef TF_TAKE
  p.total = o;
  return p;
}


// ---- JDE extensions (off on the reference path; SURVEY.md section 8 name map)
// Both phases are inlined into the extension instantiation (its own register
// allocation; the reference path never calls them): out of line, the calls
// made the caller save its live registers around them (436 B of spills, --jde
// 26.7k frames/s; inlined: 140 B, 28.7k; profiles/r02s_jde_inline_ab.txt).
// -DTF_JDE_*_ATTR=__noinline__ restores the out-of-line form.
#ifndef TF_JDE_FUSE_ATTR
#define TF_JDE_FUSE_ATTR __forceinline__
#endif
#ifndef TF_JDE_IOU_ATTR
#define TF_JDE_IOU_ATTR __forceinline__
#endif

// lambda-fused cost (JDE fuse_motion): every un-gated entry becomes
// lambda * cosine + (1 - lambda) * gate distance, the distance recomputed with
// the gate phase's arithmetic. Called by every thread of the leader; leaves
// the per-warp maxima of the fused costs in ampw[0 .. n_slots).
__device__ TF_JDE_FUSE_ATTR void fuse_motion_costs(double lambda, double lambda_w, int gate_metric, const int16_t* ecol,
                                               const int16_t* erow, double* eval, int E, const double* t_mean,
                                               const double* g_il, const double* d_meas, double* ampw, int n_slots) {
  double m = 0.0;
  for (int e = threadIdx.x; e < E; e += blockDim.x) {
    const int t = erow[e], k = ecol[e];
    const double* mu = &t_mean[8 * t];
    const double* z = &d_meas[4 * k];
    double g;
    if (gate_metric == 0) {
      g = KF::mahalanobis(mu, &g_il[4 * t], z);
    } else {
      const double dx = mu[0] - z[0], dy = mu[1] - z[1];
      g = dx * dx + dy * dy;
    }
    const double v = lambda * eval[e] + lambda_w * g;
    eval[e] = v;
    m = fmax(m, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
  if (lane_id() == 0) ampw[warp_id()] = m;
  for (int i = n_warps() + threadIdx.x; i < n_slots; i += blockDim.x) ampw[i] = 0.0;
}

// Dense rows of the second-stage matrix for the exact LAP.
struct DenseRows {
  const double* m;
  int nc;
  __device__ __forceinline__ int begin(int r) const { return r * nc; }
  __device__ __forceinline__ int end(int r) const { return r * nc + nc; }
  __device__ __forceinline__ int col(int e) const { return e % nc; }
  __device__ __forceinline__ double val(int e) const { return m[e]; }
};

// Second association stage on 1 - IoU (JDE's IoU step): tracks that were
// ACTIVE before the frame and are unmatched after the first stage, against the
// detections still unmatched, both in ascending order; boxes from the
// predicted track state and from the detections' measurements. The same exact
// solve as the first stage (sentinel padding, scipy order), then pairs above
// iou_threshold are dissolved. One warp.
__device__ TF_JDE_IOU_ATTR void iou_second_stage(double thr, int T, int K, int Tm, int Km, int cap_entries,
                                              unsigned char* smem, const double* d_meas, double* dense_global,
                                              int* err) {
  const int lane = lane_id();
  const AssocPlan pl = assoc_plan(Tm, Km, cap_entries);
  const double* t_mean = reinterpret_cast<const double*>(smem + pl.off_mean);
  const int* t_state = reinterpret_cast<const int*>(smem + pl.off_state);
  int* t_mdet = reinterpret_cast<int*>(smem + pl.off_mdet);
  double* t_mcost = reinterpret_cast<double*>(smem + pl.off_mcost);
  int* d_row = reinterpret_cast<int*>(smem + pl.off_drow);
  int16_t* rows = reinterpret_cast<int16_t*>(smem + pl.off_crows);
  int16_t* cols = reinterpret_cast<int16_t*>(smem + pl.off_ccols);
  double* dense_smem = reinterpret_cast<double*>(smem + pl.off_eval);
  const int dense_cap = cap_entries;
  LapScratch L;
  L.u = reinterpret_cast<double*>(smem + pl.off_u);
  L.v = reinterpret_cast<double*>(smem + pl.off_v);
  L.dist = reinterpret_cast<double*>(smem + pl.off_dist);
  L.crow = reinterpret_cast<double*>(smem + pl.off_crow);
  L.path = reinterpret_cast<int16_t*>(smem + pl.off_path);
  L.row4col = reinterpret_cast<int16_t*>(smem + pl.off_r4c);
  L.col4row = reinterpret_cast<int16_t*>(smem + pl.off_c4r);
  L.rem = reinterpret_cast<int16_t*>(smem + pl.off_rem);
  L.vrows = reinterpret_cast<int16_t*>(smem + pl.off_vr);
  L.vcols = reinterpret_cast<int16_t*>(smem + pl.off_vc);
  int nr = 0, nc = 0;
  for (int t0 = 0; t0 < T; t0 += 32) {                 // ordered compaction of the lists
    const int t = t0 + lane;
    const bool in = t < T && t_mdet[t] < 0 && t_state[t] == 0;
    const unsigned bm = __ballot_sync(FULL, in);
    if (in) rows[nr + __popc(bm & ((1u << lane) - 1u))] = static_cast<int16_t>(t);
    nr += __popc(bm);
  }
  for (int k0 = 0; k0 < K; k0 += 32) {
    const int k = k0 + lane;
    const bool in = k < K && d_row[k] < 0;
    const unsigned bm = __ballot_sync(FULL, in);
    if (in) cols[nc + __popc(bm & ((1u << lane) - 1u))] = static_cast<int16_t>(k);
    nc += __popc(bm);
  }
  __syncwarp();
  if (nr == 0 || nc == 0) return;
  double* dense = nr * nc <= dense_cap ? dense_smem : dense_global;
  double amp = 0.0;
  for (int x = lane; x < nr * nc; x += 32) {
    const int i = x / nc, j = x - i * nc;
    double a[4], b[4];
    const bool oka = meas_to_box(&t_mean[8 * rows[i]], a);
    const bool okb = meas_to_box(&d_meas[4 * cols[j]], b);
    if (!oka) flag_error(err, rows[i] + 1, TF_INVALID_BOX);
    if (!okb) flag_error(err, cols[j] + 1, TF_INVALID_BOX);
    const double v = 1.0 - iou_tlwh(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3]);
    dense[x] = v;
    amp = fmax(amp, fabs(v));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amp = fmax(amp, __shfl_xor_sync(FULL, amp, o));
  __syncwarp();
  const int n = nr > nc ? nr : nc;
  const double sentinel = 2.0 * static_cast<double>(n) * fmax(amp, 1.0) + 1.0;   // tf/assoc.py:67-74
  warp_lap_fast(n, nr, DenseRows{dense, nc}, sentinel, L);
  __syncwarp();
  for (int i = lane; i < nr; i += 32) {
    const int c = L.col4row[i];
    if (c < nc) {
      const double v = dense[i * nc + c];
      if (!(v > thr)) {                                   // tf/assoc.py:90-107 with the stage's threshold
        const int t = rows[i], k = cols[c];
        t_mdet[t] = k;
        t_mcost[t] = v;
        d_row[k] = t;
      }
    }
  }
  __syncwarp();
}

// Embedding rows of a frame's births, one warp per birth: each new track's
// pool slot (popped in birth order) receives its detection's embedding. Out
// of line so the row held in registers does not weigh on the kernel's
// register allocation.
__device__ __noinline__ void birth_rows(const float* dets, float* pool, const int16_t* d_pos, const int* f_stk, int nf,
                                        int K, int D) {
  const int lane = lane_id();
  for (int k = warp_id(); k < K; k += n_warps()) {
    const int r = d_pos[k];
    if (r < 0) continue;
    const float* src = dets + static_cast<long long>(k) * D;
    TF_BCHK(nf - 1 - r >= 0 && (unsigned)f_stk[nf - 1 - r] < 1024u, "birth_rows blk %d nf %d r %d slot %d\n",
            blockIdx.x, nf, r, nf - 1 - r >= 0 ? f_stk[nf - 1 - r] : -999);
    float* dst = pool + static_cast<long long>(f_stk[nf - 1 - r]) * D;
    if (D == 512) {
      float4 x[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) x[q] = reinterpret_cast<const float4*>(src)[lane + 32 * q];
#pragma unroll
      for (int q = 0; q < 4; ++q) reinterpret_cast<float4*>(dst)[lane + 32 * q] = x[q];
    } else if ((D & 3) == 0) {
      for (int i = lane; i < D / 4; i += 32) reinterpret_cast<float4*>(dst)[i] = reinterpret_cast<const float4*>(src)[i];
    } else {
      for (int i = lane; i < D; i += 32) dst[i] = src[i];
    }
  }
}

// ---- cluster-cooperative phases of associate_kernel ----------------------------
// The association of one stream is sequential per frame, but two of its phases
// are embarrassingly parallel and L2-latency bound: the fp64 cosine costs of the
// un-gated pairs and the EMA appearance updates. With a thread-block cluster per
// stream, follower CTAs join exactly these phases. Costs are statically
// partitioned over every warp of the cluster; a follower reads the entry list
// through DSMEM and sends each cost back with an asynchronous remote store
// that counts its bytes on a leader mbarrier (st.async ... complete_tx), so
// the leader's wait ends when the last cost lands, without a release fence.

// pairs per warp per round (one L2 round trip per frame where possible)
// (3 pairs when that still fits one round: more warps share a frame's
// entries; cfg1 cost phase 4.16 -> 3.98 us)
__device__ __forceinline__ int cost_nb(int E, int n_workers) {
  return E > 3 * n_workers ? 4 : E > 2 * n_workers ? 3 : 2;
}

// entries of a frame costed by follower warps (workers >= lead_workers)
__device__ __forceinline__ int follower_entries(int E, int n_workers, int lead_workers) {
  const int NB = cost_nb(E, n_workers);
  const int nblk = E / NB, rem = E - nblk * NB;
  int lead = NB * ((nblk / n_workers) * lead_workers + min(nblk % n_workers, lead_workers));
  if (rem && (nblk % n_workers) < lead_workers) lead += rem;
  return E - lead;
}

__device__ __forceinline__ void st_async_f64(unsigned cluster_addr_, double v, unsigned cluster_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];\n" ::"r"(cluster_addr_),
               "l"(__double_as_longlong(v)), "r"(cluster_bar)
               : "memory");
}

struct CostView {
  const int16_t* ecol;
  const int16_t* erow;
  double* eval;
  const int* t_slot;
  double* ampw;                // per-worker max cost (one slot per cluster warp)
  unsigned eval_cl, ampw_cl;   // leader addresses of eval / ampw for st.async ...
  unsigned bar_cl;             // ... counted on this leader mbarrier (0: plain stores)
  const float* pool;           // this stream's embedding pool
  const float* dets;           // this frame's detection embeddings
  int E, D;
};

// NB entry pairs per warp per round: every row of a round is in flight at once.
template <int NB>
__device__ __forceinline__ double cost_rounds(const CostView v, int worker, int n_workers) {
  const int lane = lane_id();
  double amp = 0.0;
  for (int e0 = NB * worker; e0 < v.E; e0 += NB * n_workers) {
    const int n = min(NB, v.E - e0);
    // remote (DSMEM) loads are issued per thread: lanes 0..NB-1 fetch the
    // detection indices, lanes NB..2NB-1 the pool slots; shuffles broadcast them
    int idx = 0;
    if (lane < 2 * NB) {
      const int e = e0 + min(lane % NB, n - 1);
      idx = lane < NB ? v.ecol[e] : v.erow[e];
      if (lane >= NB) idx = v.t_slot[idx];
    }
    int k[NB], sl[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      k[j] = __shfl_sync(FULL, idx, j);
      sl[j] = __shfl_sync(FULL, idx, NB + j);
      TF_BCHK((unsigned)sl[j] < 1024u && (unsigned)k[j] < 1024u, "cost blk %d e %d sl %d k %d\n", blockIdx.x,
              e0 + j, sl[j], k[j]);
    }
    double acc[NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) acc[j] = 0.0;
    if (v.D == 512) {
      float4 a[NB][4], b[NB][4];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const float4* x = reinterpret_cast<const float4*>(v.pool + static_cast<long long>(sl[j]) * 512);
        const float4* y = reinterpret_cast<const float4*>(v.dets + static_cast<long long>(k[j]) * 512);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          a[j][q] = x[lane + 32 * q];
          b[j][q] = y[lane + 32 * q];
        }
      }
#ifdef TF_EXPERIMENT_NOCVT
      // timing experiment only (wrong numerics): fp32 accumulation, no fp32 -> fp64 conversions
      float accf[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) accf[j] = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          accf[j] = fmaf(a[j][q].x, b[j][q].x, accf[j]);
          accf[j] = fmaf(a[j][q].y, b[j][q].y, accf[j]);
          accf[j] = fmaf(a[j][q].z, b[j][q].z, accf[j]);
          accf[j] = fmaf(a[j][q].w, b[j][q].w, accf[j]);
        }
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[j] = accf[j];
#else
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          acc[j] = fma(static_cast<double>(a[j][q].x), static_cast<double>(b[j][q].x), acc[j]);
          acc[j] = fma(static_cast<double>(a[j][q].y), static_cast<double>(b[j][q].y), acc[j]);
          acc[j] = fma(static_cast<double>(a[j][q].z), static_cast<double>(b[j][q].z), acc[j]);
          acc[j] = fma(static_cast<double>(a[j][q].w), static_cast<double>(b[j][q].w), acc[j]);
        }
#endif
    } else {
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const float* te = v.pool + static_cast<long long>(sl[j]) * v.D;
        const float* de = v.dets + static_cast<long long>(k[j]) * v.D;
        for (int i = lane; i < v.D; i += 32) acc[j] = fma(static_cast<double>(te[i]), static_cast<double>(de[i]), acc[j]);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int j = 0; j < NB; ++j) acc[j] += __shfl_xor_sync(FULL, acc[j], o);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      if (j < n) {
        const double c = fmin(fmax(1.0 - acc[j], 0.0), 2.0);
        if (lane == 0) {
          if (v.bar_cl) st_async_f64(v.eval_cl + 8u * static_cast<unsigned>(e0 + j), c, v.bar_cl);
          else v.eval[e0 + j] = c;
        }
        amp = fmax(amp, c);
      }
    }
  }
  return amp;
}

// Kept out of line: the kernel runs at the register cap, and inlining this
// phase's 2 x 4 rows of loads perturbs the allocation of every other phase.
__device__ __noinline__ void cost_work(const CostView v, int worker, int n_workers) {
  // Entry pairs are statically partitioned over every warp of the cluster
  // (worker = global warp index): no atomics on the critical path. Up to
  // 4 pairs per warp per round (4 x 2 rows x 2 KB of 128-bit loads in flight)
  // so a frame's entries take one round trip to L2 where possible.
  const int nb = cost_nb(v.E, n_workers);
  const double amp = nb == 4   ? cost_rounds<4>(v, worker, n_workers)
                     : nb == 3 ? cost_rounds<3>(v, worker, n_workers)
                               : cost_rounds<2>(v, worker, n_workers);
  // amplitude = max |finite| (tf/assoc.py:71): one slot per worker, reduced
  // by the leader (a contended u64 atomicMax over DSMEM is a CAS loop)
  if (lane_id() == 0) {
    if (v.bar_cl) st_async_f64(v.ampw_cl + 8u * static_cast<unsigned>(worker), amp, v.bar_cl);
    else v.ampw[worker] = amp;
  }
}

struct EmaView {
  const int* slot;             // pool slot of each detection's matched track, -1 if none
  int* work;
  int* err;
  float* pool;
  const float* dets;
  double alpha, beta;
  int K, D;
};

// One matched detection's EMA from rows already in registers (D = 512):
// normalize(alpha * old + beta * new) in fp64, fp32 out.
__device__ __forceinline__ void ema_row512(const EmaView& v, int k, int sl, const float4 (&x)[4], const float4 (&y)[4]) {
  const int lane = lane_id();
  double w[16];
  double ss = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    w[4 * q + 0] = v.alpha * static_cast<double>(x[q].x) + v.beta * static_cast<double>(y[q].x);
    w[4 * q + 1] = v.alpha * static_cast<double>(x[q].y) + v.beta * static_cast<double>(y[q].y);
    w[4 * q + 2] = v.alpha * static_cast<double>(x[q].z) + v.beta * static_cast<double>(y[q].z);
    w[4 * q + 3] = v.alpha * static_cast<double>(x[q].w) + v.beta * static_cast<double>(y[q].w);
  }
#pragma unroll
  for (int q = 0; q < 16; ++q) ss = fma(w[q], w[q], ss);
  ss = warp_sum(ss);
  const double nrm = sqrt(ss);
  if (!(nrm >= 1e-12) || !isfinite(nrm)) {
    if (lane == 0) flag_error(v.err, k + 1, TF_DEGENERATE_EMBEDDING);
    return;
  }
  float4* o4 = reinterpret_cast<float4*>(v.pool + static_cast<long long>(sl) * 512);
  const double rn = __drcp_rn(nrm);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    float4 r;
    r.x = static_cast<float>(div_by(w[4 * q + 0], nrm, rn));
    r.y = static_cast<float>(div_by(w[4 * q + 1], nrm, rn));
    r.z = static_cast<float>(div_by(w[4 * q + 2], nrm, rn));
    r.w = static_cast<float>(div_by(w[4 * q + 3], nrm, rn));
    o4[lane + 32 * q] = r;
  }
}

// EMA appearance update (tf/tracker.py:67-71, 117-119): one warp per matched
// detection, normalize(alpha * old + (1 - alpha) * new) in fp64, fp32 out.
// D = 512: a warp claims two detections at a time and has both pairs of rows
// in flight before it computes either (one round trip per two items).
__device__ void ema_work(const EmaView v) {
  const int lane = lane_id();
#ifndef TF_EMA_SINGLE
  if (v.D == 512) {
    // two detections per claim: the second's rows are prefetched into L1
    // while the first is computed, so its loads do not wait a round trip
    for (;;) {
      int k0 = 0;
      if (lane == 0) k0 = atomicAdd(v.work, 2);
      k0 = __shfl_sync(FULL, k0, 0);
      if (k0 >= v.K) return;
      int s0 = -1, s1 = -1;
      if (lane == 0) {
        s0 = v.slot[k0];
        s1 = k0 + 1 < v.K ? v.slot[k0 + 1] : -1;
      }
      s0 = __shfl_sync(FULL, s0, 0);
      s1 = __shfl_sync(FULL, s1, 0);
      if (s1 >= 0) {
        const float* t = v.pool + static_cast<long long>(s1) * 512;
        const float* d = v.dets + static_cast<long long>(k0 + 1) * 512;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          asm volatile("prefetch.global.L1 [%0];" ::"l"(t + 4 * (lane + 32 * q)));
          asm volatile("prefetch.global.L1 [%0];" ::"l"(d + 4 * (lane + 32 * q)));
        }
      }
#pragma unroll 1
      for (int i = 0; i < 2; ++i) {
        const int k = k0 + i, sl = i ? s1 : s0;
        if (sl < 0) continue;
        const float4* t4 = reinterpret_cast<const float4*>(v.pool + static_cast<long long>(sl) * 512);
        const float4* d4 = reinterpret_cast<const float4*>(v.dets + static_cast<long long>(k) * 512);
        float4 x[4], y[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) { x[q] = t4[lane + 32 * q]; y[q] = d4[lane + 32 * q]; }
        ema_row512(v, k, sl, x, y);
      }
    }
  }
#endif
  for (;;) {
    int k = 0;
    if (lane == 0) k = atomicAdd(v.work, 1);
    k = __shfl_sync(FULL, k, 0);
    if (k >= v.K) break;
    int sl = 0;
    if (lane == 0) sl = v.slot[k];           // one remote load, broadcast
    sl = __shfl_sync(FULL, sl, 0);
    if (sl < 0) continue;
    TF_BCHK((unsigned)sl < 1024u, "ema blk %d k %d sl %d\n", blockIdx.x, k, sl);
    float* te = v.pool + static_cast<long long>(sl) * v.D;
    const float* de = v.dets + static_cast<long long>(k) * v.D;
    if (v.D == 512) {                                   // one pass, rows held in registers
      const float4* t4 = reinterpret_cast<const float4*>(te);
      const float4* d4 = reinterpret_cast<const float4*>(de);
      float4 x[4], y[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { x[q] = t4[lane + 32 * q]; y[q] = d4[lane + 32 * q]; }
      double w[16];
      double ss = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        w[4 * q + 0] = v.alpha * static_cast<double>(x[q].x) + v.beta * static_cast<double>(y[q].x);
        w[4 * q + 1] = v.alpha * static_cast<double>(x[q].y) + v.beta * static_cast<double>(y[q].y);
        w[4 * q + 2] = v.alpha * static_cast<double>(x[q].z) + v.beta * static_cast<double>(y[q].z);
        w[4 * q + 3] = v.alpha * static_cast<double>(x[q].w) + v.beta * static_cast<double>(y[q].w);
      }
#pragma unroll
      for (int q = 0; q < 16; ++q) ss = fma(w[q], w[q], ss);
      ss = warp_sum(ss);
      const double nrm = sqrt(ss);
      if (!(nrm >= 1e-12) || !isfinite(nrm)) {
        if (lane == 0) flag_error(v.err, k + 1, TF_DEGENERATE_EMBEDDING);
        continue;
      }
      float4* o4 = reinterpret_cast<float4*>(te);
      const double rn = __drcp_rn(nrm);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float4 r;
        r.x = static_cast<float>(div_by(w[4 * q + 0], nrm, rn));
        r.y = static_cast<float>(div_by(w[4 * q + 1], nrm, rn));
        r.z = static_cast<float>(div_by(w[4 * q + 2], nrm, rn));
        r.w = static_cast<float>(div_by(w[4 * q + 3], nrm, rn));
        o4[lane + 32 * q] = r;
      }
      continue;
    }
    double ss = 0.0;
    for (int i = lane; i < v.D; i += 32) {
      double w = v.alpha * static_cast<double>(te[i]) + v.beta * static_cast<double>(de[i]);
      ss = fma(w, w, ss);
    }
    ss = warp_sum(ss);
    const double nrm = sqrt(ss);
    if (!(nrm >= 1e-12) || !isfinite(nrm)) {
      if (lane == 0) flag_error(v.err, k + 1, TF_DEGENERATE_EMBEDDING);
      continue;
    }
    __syncwarp();
    for (int i = lane; i < v.D; i += 32) {
      double w = v.alpha * static_cast<double>(te[i]) + v.beta * static_cast<double>(de[i]);
      te[i] = static_cast<float>(w / nrm);
    }
  }
}

// Cluster hand-offs of a frame. Leader -> followers (entries ready, EMA list
// published): the hardware cluster barrier, the leader arriving with release
// semantics and waiting for the phase only before its next arrive; the
// scalars a follower needs are pushed into its shared memory first.
// Followers -> leader: costs arrive by st.async on a transaction-counting
// mbarrier; the EMA of a frame, applied while the leader runs on, is
// signalled by one release arrive per follower on another leader mbarrier.
__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ unsigned cluster_addr(const void* p, unsigned rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(unsigned cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void st_cluster(unsigned cluster_addr_, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;\n" ::"r"(cluster_addr_), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "TF_MBAR_WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra TF_MBAR_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// kThreads = 256: one CTA per SM (the register file is the limit), clusters
// for few streams. kThreads = 128: two CTAs per SM for launches with more
// streams than twice the SM count (the host halves the shared-memory plan).
// kExt: the JDE extensions (lambda-fused cost, IoU second stage) are compiled
// only into their own instantiations, so the reference path keeps its code.
// Longest-processing-time-first order of n single-CTA streams for the next
// launch over the same streams, from this launch's per-stream work (cycles of
// the frame loop): a counting sort into 1024 buckets, heaviest bucket first.
// Order inside a bucket is arbitrary (it only steers the block scheduler; the
// results do not depend on it). Run by the last CTA to finish; scratch: 2048
// ints of shared memory.
__device__ void lpt_order(const long long* work, int* order, int n, int* scratch) {
  constexpr int kBuckets = 1024;
  int* hist = scratch;
  int* off = scratch + kBuckets;
  __shared__ long long s_lo, s_hi;
  const int tid = threadIdx.x;
  if (tid == 0) { s_lo = LLONG_MAX; s_hi = LLONG_MIN; }
  for (int i = tid; i < kBuckets; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  long long lo = LLONG_MAX, hi = LLONG_MIN;
  for (int i = tid; i < n; i += blockDim.x) {
    const long long w = __ldcg(work + i);
    lo = min(lo, w);
    hi = max(hi, w);
  }
  atomicMin(reinterpret_cast<long long*>(&s_lo), lo);
  atomicMax(reinterpret_cast<long long*>(&s_hi), hi);
  __syncthreads();
  const double span = static_cast<double>(s_hi - s_lo) + 1.0;
  auto bucket = [&](int i) {
    const int b = static_cast<int>(static_cast<double>(s_hi - __ldcg(work + i)) * (kBuckets - 1) / span);
    return min(max(b, 0), kBuckets - 1);
  };
  for (int i = tid; i < n; i += blockDim.x) atomicAdd(&hist[bucket(i)], 1);
  __syncthreads();
  if (tid < 32) {                             // exclusive scan of the histogram by one warp
    int run = 0;
    for (int c = 0; c < kBuckets; c += 32) {
      const int v = hist[c + tid];
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(FULL, x, o);
        if (tid >= o) x += y;
      }
      off[c + tid] = run + x - v;
      run += __shfl_sync(FULL, x, 31);
    }
  }
  __syncthreads();
  for (int i = tid; i < n; i += blockDim.x) order[atomicAdd(&off[bucket(i)], 1)] = i;
}

template <int kThreads, bool kExt>
__global__ void __launch_bounds__(kThreads, 256 / kThreads) associate_kernel(AssocArgs a, Params P) {
  extern __shared__ __align__(16) unsigned char smem[];
  const long long t_k0 = clock64();           // launch prologue / epilogue timers (slots 28, 29)
  auto gtimer = [] { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; };
  const int C = a.cluster;                   // CTAs per stream (thread-block cluster)
  int ls = blockIdx.x / C;                   // local stream in this update (a.order_in: see below)
  int s = a.stream_begin + ls;               // global stream id
  const int rank = C > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
  const int tid = threadIdx.x, lane = lane_id(), wid = warp_id(), nw = n_warps();
  long long t_gt0 = 0;
  if (a.sclk && tid == 0 && rank == 0) t_gt0 = gtimer();
  const int Tm = a.cap_tracks, Km = a.cap_det, D = P.dim;
  const int KW = (Km + 31) / 32;
  const AssocPlan pl = assoc_plan(Tm, Km, a.cap_entries);
  int64_t* t_id = reinterpret_cast<int64_t*>(smem + pl.off_id);
  int64_t* t_lost = reinterpret_cast<int64_t*>(smem + pl.off_lost);
  int64_t* t_last = reinterpret_cast<int64_t*>(smem + pl.off_last);
  double* t_mean = reinterpret_cast<double*>(smem + pl.off_mean);
  double* t_cov = reinterpret_cast<double*>(smem + pl.off_cov);
  double* t_mcost = reinterpret_cast<double*>(smem + pl.off_mcost);
  int* t_state = reinterpret_cast<int*>(smem + pl.off_state);
  int* t_hits = reinterpret_cast<int*>(smem + pl.off_hits);
  int* t_slot = reinterpret_cast<int*>(smem + pl.off_slot);
  int* t_mdet = reinterpret_cast<int*>(smem + pl.off_mdet);
  int* rowptr = reinterpret_cast<int*>(smem + pl.off_rowptr);
  int* t_flag = reinterpret_cast<int*>(smem + pl.off_flag);
  int16_t* npos = reinterpret_cast<int16_t*>(smem + pl.off_npos);
  int16_t* rpos = reinterpret_cast<int16_t*>(smem + pl.off_rpos);
  double* const d_meas0 = reinterpret_cast<double*>(smem + pl.off_dm);
  double* const d_obj0 = reinterpret_cast<double*>(smem + pl.off_dobj);
  double* const d_meas1 = reinterpret_cast<double*>(smem + pl.off_dm2);
  double* const d_obj1 = reinterpret_cast<double*>(smem + pl.off_dobj2);
  double* d_meas = d_meas0;
  double* d_obj = d_obj0;
  int* d_row = reinterpret_cast<int*>(smem + pl.off_drow);
  int16_t* d_pos = reinterpret_cast<int16_t*>(smem + pl.off_dpos);
  unsigned* gmask = reinterpret_cast<unsigned*>(smem + pl.off_gmask);
  double* g_il = reinterpret_cast<double*>(smem + pl.off_il);   // 1/sqrt(S_i) per track (gate phase)
  LapScratch L;
  L.u = reinterpret_cast<double*>(smem + pl.off_u);
  L.v = reinterpret_cast<double*>(smem + pl.off_v);
  L.dist = reinterpret_cast<double*>(smem + pl.off_dist);
  L.crow = reinterpret_cast<double*>(smem + pl.off_crow);
  L.path = reinterpret_cast<int16_t*>(smem + pl.off_path);
  L.row4col = reinterpret_cast<int16_t*>(smem + pl.off_r4c);
  L.col4row = reinterpret_cast<int16_t*>(smem + pl.off_c4r);
  L.rem = reinterpret_cast<int16_t*>(smem + pl.off_rem);
  L.vrows = reinterpret_cast<int16_t*>(smem + pl.off_vr);
  L.vcols = reinterpret_cast<int16_t*>(smem + pl.off_vc);
  int* c_lab = reinterpret_cast<int*>(smem + pl.off_lab);
  int* c_nr = reinterpret_cast<int*>(smem + pl.off_cnr);
  int* c_nc = reinterpret_cast<int*>(smem + pl.off_cnc);
  int* c_ne = reinterpret_cast<int*>(smem + pl.off_cne);
  int* c_root = reinterpret_cast<int*>(smem + pl.off_croot);
  int* c_off = reinterpret_cast<int*>(smem + pl.off_coff);
  int16_t* c_pos = reinterpret_cast<int16_t*>(smem + pl.off_cpos);
  int16_t* c_rows = reinterpret_cast<int16_t*>(smem + pl.off_crows);
  int16_t* c_cols = reinterpret_cast<int16_t*>(smem + pl.off_ccols);
  int16_t* c_map = reinterpret_cast<int16_t*>(smem + pl.off_cmap);
  int16_t* rcol = reinterpret_cast<int16_t*>(smem + pl.off_rcol);
  int16_t* const smem_epos = reinterpret_cast<int16_t*>(smem + pl.off_epos);
  int16_t* c_epos = smem_epos;
  int16_t* c_rmap = reinterpret_cast<int16_t*>(smem + pl.off_rmap);
  int* c_lrp = reinterpret_cast<int*>(smem + pl.off_lrp);
  int* c_eoff = reinterpret_cast<int*>(smem + pl.off_eoff);
  int16_t* const smem_elist = reinterpret_cast<int16_t*>(smem + pl.off_elist);
  int16_t* c_elist = smem_elist;
  unsigned long long* p_cmin = reinterpret_cast<unsigned long long*>(smem + pl.off_pcmin);
  double* p_rmin = reinterpret_cast<double*>(smem + pl.off_prmin);
  int* p_ccnt = reinterpret_cast<int*>(smem + pl.off_pccnt);
  int* p_cdeg = reinterpret_cast<int*>(smem + pl.off_pcdeg);
  int* p_crow = reinterpret_cast<int*>(smem + pl.off_pcrow);
  int* p_rdeg = reinterpret_cast<int*>(smem + pl.off_prdeg);
  int* p_rcnt = reinterpret_cast<int*>(smem + pl.off_prcnt);
  int* p_rc1 = reinterpret_cast<int*>(smem + pl.off_prc1);
  uint8_t* p_ra = smem + pl.off_pra;
  uint8_t* p_ca = smem + pl.off_pca;
  uint8_t* p_kr = smem + pl.off_pkr;
  uint8_t* p_kc = smem + pl.off_pkc;
  if (a.zero_smem) {            // diagnostics: no byte of the plan keeps a previous CTA's value
    for (size_t x = threadIdx.x; x < pl.total / 16; x += blockDim.x) reinterpret_cast<uint4*>(smem)[x] = make_uint4(0, 0, 0, 0);
    __syncthreads();
  }
  for (int x = threadIdx.x; x < Tm; x += blockDim.x) p_kr[x] = 0;
  for (int x = threadIdx.x; x < Km; x += blockDim.x) p_kc[x] = 0;

  __shared__ int s_warp[33];
  __shared__ unsigned long long s_scan64[33];
  __shared__ int s_T, s_status, s_E, s_nfree, s_err, s_flag, s_tie, s_Efr;
  __shared__ int s_alt;     // a component solve found a near-optimum (written only after every thread read s_tie)
  __shared__ int s_ema_work, s_ema_err, s_ema_b, s_flag2, s_nlive[2], s_nmulti;
  __shared__ int s_cflag;   // component labelling (its own flag: threads may still be reading peeling's last s_flag)   // the follower-applied EMA of frame s_ema_b
  int* ema_slot = reinterpret_cast<int*>(smem + pl.off_emas);
  int* f_stk = reinterpret_cast<int*>(smem + pl.off_fstk);

  // optional phase timing (tf_set_profiling): cycles per phase + counters
  __shared__ long long s_ph[kPhaseSlots];
  long long t_mark = 0, t_sub = 0;
#define TF_SUB(i)                                     \
  if (a.stats && tid == 0) {                          \
    const long long now_ = clock64();                 \
    s_ph[(i)] += now_ - t_sub;                        \
    t_sub = now_;                                     \
  }
#ifdef TF_CANARY
  // debug: 64 words past the plan, checked at every phase mark (smem overrun hunt)
  unsigned* const canary = reinterpret_cast<unsigned*>(smem + pl.total);
  for (int x = tid; x < 64; x += blockDim.x) canary[x] = 0xC0FFEE00u + x;
#define TF_CANARY_CHECK(i)                                                                          \
  if (tid == 0)                                                                                     \
    for (int x_ = 0; x_ < 64; ++x_)                                                                 \
      if (canary[x_] != 0xC0FFEE00u + x_) {                                                         \
        printf("TFCANARY blk %d frame %d mark %d word %d val %08x\n", blockIdx.x, b, (i), x_, canary[x_]); \
        canary[x_] = 0xC0FFEE00u + x_;                                                              \
      }
#else
#define TF_CANARY_CHECK(i)
#endif
#define TF_MARK(i)                                    \
  TF_CANARY_CHECK(i)                                  \
  if (a.stats && tid == 0) {                          \
    const long long now_ = clock64();                 \
    if ((i) > 0) s_ph[(i)] += now_ - t_mark;          \
    else s_ph[0] += now_ - t_frame0;                  \
    t_mark = now_;                                    \
    t_sub = now_;                                     \
  }
  long long t_frame0 = 0;
  for (int x = tid; x < kPhaseSlots; x += blockDim.x) s_ph[x] = 0;
  __shared__ long long s_next;
  __shared__ double s_amp;
  __shared__ double s_ampw[128];    // per-worker cost maxima (cluster warps <= 128)

  // Large-E overflow: entries go to this stream's global pool.
  int16_t* const smem_ecol = reinterpret_cast<int16_t*>(smem + pl.off_ecol);
  int16_t* const smem_erow = reinterpret_cast<int16_t*>(smem + pl.off_erow);
  double* const smem_eval = reinterpret_cast<double*>(smem + pl.off_eval);
  int16_t* ecol = smem_ecol;
  int16_t* erow = smem_erow;
  double* eval = smem_eval;

  // Leader mbarriers: [0] EMA applied (C - 1 follower release arrivals),
  // [1] costs landed (leader arrive + expected st.async bytes), [2] costs
  // written to the global pool (C - 1 follower release arrivals; frames
  // whose entries overflow shared memory). The leader pushes the scalars a
  // follower needs into its s_fl before each cluster-barrier release:
  // {stop, E, T, K of the EMA list}.
  __shared__ __align__(8) unsigned long long s_bar[3];
  __shared__ __align__(16) int s_fl[4];
  if (C > 1) {
    if (tid == 0 && rank == 0) {
      mbar_init(&s_bar[0], C - 1);
      mbar_init(&s_bar[1], 1);
      mbar_init(&s_bar[2], C - 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    cg::this_cluster().sync();
  }
  // Programmatic dependent launch: the next association launch on this
  // stream may be scheduled now and run its set-up (above) while this one
  // works; it waits here for this grid's completion (and its memory) before
  // touching the track tables and embedding pool that this launch writes.
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
  // Overlapped mode (a.ready): the preceding grid is the decode of this very
  // update; frames are awaited one by one on its ready flags (below) instead
  // of on its completion. The track tables were written by the association
  // before that decode grid, which had completed when the decode grid began.
  if (a.ready == nullptr) asm volatile("griddepcontrol.wait;\n" ::: "memory");
  // Longest-first stream order (single-CTA streams over more than one wave):
  // the previous launch over these streams ranked them by its measured work
  // (lpt_order below), so the heaviest streams take the first wave and the
  // light ones fill the slots that free up. Read only after the wait above:
  // the previous launch wrote it.
  if (a.order_in) {
    ls = a.order_in[blockIdx.x];
    s = a.stream_begin + ls;
  }
  if (a.sclk && tid == 0 && rank == 0) a.sclk[4 * s] = t_gt0;

  if (rank != 0) {
    // ---- follower CTA: joins the cost and EMA phases of every frame -------
    cg::cluster_group cl = cg::this_cluster();
    const unsigned L_ema_done = cluster_addr(&s_bar[0], 0);
    const unsigned L_cost_tx = cluster_addr(&s_bar[1], 0);
    const unsigned L_cost_pool = cluster_addr(&s_bar[2], 0);
    const long long sTf = static_cast<long long>(s) * Tm;
    for (int b = 0;; ++b) {
      cluster_arrive_relaxed();                                        // S1: entries ready
      cluster_wait_acquire();
      if (s_fl[0]) return;                                             // stop: nothing of ours is read any more
      const long long fKf = static_cast<long long>(ls * a.B + b) * Km;
      const int E = s_fl[1];
      const bool pooled = E > a.cap_entries;
      if (E > 0) {
        CostView cv;
        cv.ecol = pooled ? a.pool_col + static_cast<long long>(s) * Tm * Km : cl.map_shared_rank(smem_ecol, 0);
        cv.erow = pooled ? a.pool_row + static_cast<long long>(s) * Tm * Km : cl.map_shared_rank(smem_erow, 0);
        cv.eval = pooled ? a.pool_val + static_cast<long long>(s) * Tm * Km : nullptr;
        cv.t_slot = cl.map_shared_rank(t_slot, 0);
        cv.ampw = cl.map_shared_rank(s_ampw, 0);
        cv.eval_cl = cluster_addr(smem_eval, 0);
        cv.ampw_cl = cluster_addr(s_ampw, 0);
        cv.bar_cl = pooled ? 0u : L_cost_tx;
        cv.pool = a.trk.emb_pool + sTf * static_cast<long long>(D);
        cv.dets = a.det.emb + fKf * static_cast<long long>(D);
        cv.E = E;
        cv.D = D;
        cost_work(cv, rank * n_warps() + warp_id(), n_warps() * C);
        if (pooled) {                                                  // S2 (pooled): costs written
          __syncthreads();
          if (tid == 0) mbar_arrive_remote(L_cost_pool);
        }
      }
      cluster_arrive_relaxed();                                        // S3: EMA list published
      cluster_wait_acquire();
      // The EMA of frame b runs while the leader finishes frame b and starts
      // frame b + 1; the leader waits for it before releasing that frame's costs.
      const int Ke = s_fl[3];
      if (Ke > 0) {
        EmaView ev;
        ev.slot = cl.map_shared_rank(ema_slot, 0);
        ev.work = cl.map_shared_rank(&s_ema_work, 0);
        ev.err = cl.map_shared_rank(&s_ema_err, 0);
        ev.pool = a.trk.emb_pool + sTf * static_cast<long long>(D);
        ev.dets = a.det.emb + fKf * static_cast<long long>(D);
        ev.alpha = P.alpha;
        ev.beta = P.beta;
        ev.K = Ke;
        ev.D = D;
        ema_work(ev);
      }
      __syncthreads();
      if (tid == 0) mbar_arrive_remote(L_ema_done);                    // EMA applied
    }
  }
  if (tid == 0) { s_ema_err = STATUS_CLEAR; s_ema_b = -1; }
  bool ema_out = false;           // followers may still be applying an EMA list
  bool s3_pending = false;        // the leader arrived at S3 and has not waited for the phase
  bool s1_done = false;           // this frame's S1 arrive already issued (frames with entries)
  unsigned ph_ema_done = 0, ph_cost_tx = 0, ph_cost_pool = 0;
  // lane j of warp 0 pushes follower j + 1's scalars
  const bool signaller = C > 1 && wid == 0 && lane < C - 1;
  const unsigned F_fl = signaller ? cluster_addr(s_fl, lane + 1) : 0u;
  TrackBuf& tb = a.trk;
  const long long sT = static_cast<long long>(s) * Tm;
  if (tid == 0) {
    s_T = tb.n_tracks[s];
    s_next = tb.next_id[s];
    s_nfree = tb.n_free[s];
    s_status = 0;
  }
  __syncthreads();
  int T = s_T;
  for (int t = tid; t < T; t += blockDim.x) {
    t_id[t] = tb.id[sT + t];
    t_lost[t] = tb.lost[sT + t];
    t_last[t] = tb.last[sT + t];
    t_state[t] = tb.state[sT + t];
    t_hits[t] = tb.hits[sT + t];
    t_slot[t] = tb.slot[sT + t];
    for (int q = 0; q < 8; ++q) t_mean[8 * t + q] = tb.mean[(sT + t) * 8 + q];
    for (int q = 0; q < 12; ++q) t_cov[12 * t + q] = tb.cov[(sT + t) * 12 + q];
  }
  for (int i = tid; i < s_nfree; i += blockDim.x) f_stk[i] = tb.free_stack[sT + i];
  // frame table of the update (index, decode status, detection count) and
  // the first frame's detections: the per-frame scalar loads and the
  // measurement copy leave the frame's critical path
  __shared__ long long s_fidx[kFrameTable];
  __shared__ int s_fst[kFrameTable], s_fcnt[kFrameTable];
  const bool await_frames = a.ready != nullptr;   // overlapped mode: frames arrive while this CTA runs
  for (int i = tid; i < a.B && i < kFrameTable; i += blockDim.x) {
    const int fi = ls * a.B + i;
    s_fidx[i] = fi < a.n_fidx_inline ? a.fidx_inline[fi] : a.frame_index[fi];
    if (!await_frames) {
      s_fst[i] = a.det.status[fi];
      s_fcnt[i] = min(a.det.count[fi], Km);
    }
  }
  // overlapped mode: thread 0 waits for frame b's ready flag (acquire) and
  // stages its scalars; polls frame b + 1 (its prefetch is issued only if it
  // is already decoded). The caller's barrier publishes both to the CTA.
  __shared__ int s_next_ready;
  auto await_frame = [&](int b) {
    const int fi = ls * a.B + b;
    while (ld_acquire_gpu(a.ready + fi) != a.epoch) __nanosleep(256);
    if (b < kFrameTable) {
      s_fst[b] = a.det.status[fi];
      s_fcnt[b] = min(a.det.count[fi], Km);
    }
    int nr = 0;
    if (b + 1 < a.B && ld_acquire_gpu(a.ready + fi + 1) == a.epoch) {
      nr = 1;
      if (b + 1 < kFrameTable) {
        s_fst[b + 1] = a.det.status[fi + 1];
        s_fcnt[b + 1] = min(a.det.count[fi + 1], Km);
      }
    }
    s_next_ready = nr;
  };
  auto frame_count = [&](int b) { return b < kFrameTable ? s_fcnt[b] : min(a.det.count[ls * a.B + b], Km); };
  auto prefetch_dets = [&](int b, double* dm, double* dob) {
    // cp.async (LDGSTS): 2 x 16 B of measurement + 8 B objectness per detection
    const long long fKp = static_cast<long long>(ls * a.B + b) * Km;
    const int Kp = frame_count(b);
    for (int k = tid; k < Kp; k += blockDim.x) {
      const double* sm = a.det.meas + (fKp + k) * 4;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dm + 4 * k)), "l"(sm) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dm + 4 * k + 2)), "l"(sm + 2) : "memory");
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(dob + k)), "l"(a.det.obj + fKp + k) : "memory");
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  __syncthreads();
  if (a.B > 0 && !await_frames) prefetch_dets(0, d_meas0, d_obj0);
  bool have_dets = !await_frames;   // this frame's detections were prefetched

  long long t_top = 0;
  if (a.stats && tid == 0) s_ph[28] += clock64() - t_k0;
  if (a.sclk && tid == 0) a.sclk[4 * s + 1] = gtimer();
  const long long t_work0 = clock64();
  long long t_epi = 0;
  for (int b = 0; b < a.B; ++b) {
    if (a.stats && tid == 0) {                     // whole-frame cycles (slot 31)
      const long long now_ = clock64();
      if (b > 0) s_ph[31] += now_ - t_top;
      t_top = now_;
    }
    if (s_status != 0) break;                      // stream failed earlier: stop
    if (await_frames) {
      if (tid == 0) await_frame(b);
      __syncthreads();
      if (!have_dets) prefetch_dets(b, (b & 1) ? d_meas1 : d_meas0, (b & 1) ? d_obj1 : d_obj0);
    }
    const int f = ls * a.B + b;
    const long long fK = static_cast<long long>(f) * Km;
    const long long frame = b < kFrameTable ? s_fidx[b] : f < a.n_fidx_inline ? a.fidx_inline[f] : a.frame_index[f];
    const int fst = b < kFrameTable ? s_fst[b] : a.det.status[f];
    if (fst != 0) {                                // decode/NMS error of this frame
      if (tid == 0) s_status = (b << 8) | fst;
      break;
    }
    const int K = frame_count(b);
    T = s_T;
    TF_BCHK(tid != 0 || (T + s_nfree == Tm && T <= Tm && K <= Km), "frame blk %d b %d T %d nfree %d Tm %d K %d\n",
            blockIdx.x, b, T, s_nfree, Tm, K);
    TF_XSYNC(0);
    if (tid == 0) { s_err = STATUS_CLEAR; s_amp = 0.0; s_Efr = 0; t_frame0 = clock64(); }
    // this frame's detections were prefetched (this thread's copies land here;
    // the predict barrier publishes all of them); start the next frame's
    d_meas = (b & 1) ? d_meas1 : d_meas0;
    d_obj = (b & 1) ? d_obj1 : d_obj0;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    have_dets = b + 1 < a.B && (!await_frames || s_next_ready);
    if (have_dets) prefetch_dets(b + 1, (b & 1) ? d_meas0 : d_meas1, (b & 1) ? d_obj0 : d_obj1);
    for (int k = tid; k < K; k += blockDim.x) d_row[k] = -1;
    // ---- Kalman predict for every live track (tf/tracker.py:98-99) --------
    const bool gating = (T > 0 && K > 0);
    for (int t = tid; t < T; t += blockDim.x) {
      double* m = &t_mean[8 * t];
      double* c = &t_cov[12 * t];
      KF::predict(P, m, c);
      t_mdet[t] = -1;
      t_flag[t] = 0;
      if (gating && P.gate_metric == 0) {
        double sv[4];
        if (!KF::project(P, m, c, sv, &g_il[4 * t])) flag_error(&s_err, t + 1, TF_NUMERIC);
      }
    }
    if (tid == 0 && gating && P.gate_metric != 0 && P.gate_metric != 1) flag_error(&s_err, 0, TF_CONFIG);
    __syncthreads();
    TF_MARK(0);

    // ---- gate (tf/tracker.py:109-110, tf/motion.py:128-142) ----------------
    // Each warp takes four tracks at a time and walks the detection chunks
    // (lanes own detections). The four fp64 chains are branch-free (rows past
    // T are clamped and masked) so they interleave; the per-track count is a
    // plain store, no atomics.
    if (gating) {
      const int KC = (K + 31) >> 5;
      const double thr = P.gate_threshold;
      const bool maha = (P.gate_metric == 0);
#ifndef TF_GU
#define TF_GU 6
#endif
      constexpr int GU = TF_GU;            // tracks per warp pass (independent fp64 chains; 6: -0.12 us/frame vs 4; 3, 7, 8 slower)
      for (int t0 = GU * wid; t0 < T; t0 += GU * nw) {
        int cnt[GU];
#pragma unroll
        for (int u = 0; u < GU; ++u) cnt[u] = 0;
        for (int kc = 0; kc < KC; ++kc) {
          const int k = (kc << 5) + lane;
          const int kk = min(k, K - 1);
          const double z0 = d_meas[4 * kk], z1 = d_meas[4 * kk + 1], z2 = d_meas[4 * kk + 2], z3 = d_meas[4 * kk + 3];
          double g[GU];
#pragma unroll
          for (int u = 0; u < GU; ++u) {
            const int t = min(t0 + u, T - 1);
            const double* m = &t_mean[8 * t];
            if (maha) {
              const double* il = &g_il[4 * t];
              const double x0 = (z0 - m[0]) * il[0];
              const double x1 = (z1 - m[1]) * il[1];
              const double x2 = (z2 - m[2]) * il[2];
              const double x3 = (z3 - m[3]) * il[3];
              g[u] = ((x0 * x0 + x1 * x1) + x2 * x2) + x3 * x3;
            } else {
              const double dx = m[0] - z0, dy = m[1] - z1;
              g[u] = dx * dx + dy * dy;
            }
          }
#pragma unroll
          for (int u = 0; u < GU; ++u) {
            const bool fin = k < K && t0 + u < T && !(g[u] > thr);
            const unsigned bm = __ballot_sync(FULL, fin);
            cnt[u] += __popc(bm);
            if (lane == 0 && t0 + u < T) gmask[(t0 + u) * KW + kc] = bm;
          }
        }
        if (lane == 0) {
#pragma unroll
          for (int u = 0; u < GU; ++u)
            if (t0 + u < T) t_flag[t0 + u] = cnt[u];
        }
      }
    }
    __syncthreads();
    TF_MARK(1);
    // ---- CSR of finite (un-gated) entries, row-major -----------------------
    if (gating) {
      if (wid == 0) {                    // lanes own 4 consecutive rows per pass
        int carry = 0;
        for (int t0 = 0; t0 < T; t0 += 128) {
          int v[4], sum = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = t0 + 4 * lane + j;
            v[j] = t < T ? t_flag[t] : 0;
            sum += v[j];
          }
          int incl = sum;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            int q = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += q;
          }
          int run = carry + incl - sum;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int t = t0 + 4 * lane + j;
            if (t < T) rowptr[t] = run;
            run += v[j];
          }
          carry += __shfl_sync(FULL, incl, 31);
        }
        if (lane == 0) { rowptr[T] = carry; s_E = carry; }
      }
      __syncthreads();
      const int E = s_E;
      // entry storage is chosen per frame (follower CTAs make the same choice)
      const bool pooled = E > a.cap_entries;
      ecol = pooled ? a.pool_col + static_cast<long long>(s) * Tm * Km : smem_ecol;
      erow = pooled ? a.pool_row + static_cast<long long>(s) * Tm * Km : smem_erow;
      eval = pooled ? a.pool_val + static_cast<long long>(s) * Tm * Km : smem_eval;
      c_epos = pooled ? a.pool_aux + static_cast<long long>(s) * 2 * Tm * Km : smem_epos;
      c_elist = pooled ? a.pool_aux + static_cast<long long>(s) * 2 * Tm * Km + static_cast<long long>(Tm) * Km
                       : smem_elist;
      // one thread per (row, mask word): its entries start after the row's
      // earlier words
      const int KWf = (K + 31) >> 5;
      for (int x = tid; x < T * KWf; x += blockDim.x) {
        const int t = x / KWf, w = x - t * KWf;
        const unsigned* row = &gmask[t * KW];
        int e = rowptr[t];
        for (int w2 = 0; w2 < w; ++w2) e += __popc(row[w2]);
        unsigned bm = row[w];
        while (bm) {
          const int b = __ffs(bm) - 1;
          bm &= bm - 1u;
          ecol[e] = static_cast<int16_t>(w * 32 + b);
          erow[e] = static_cast<int16_t>(t);
          ++e;
        }
      }
      if (C > 1) {
        // S1 straight after this thread's share of the scatter: the
        // release's fence overlaps the other warps' scatter work (-0.4 us
        // per frame against arriving after the CTA barrier)
        if (s3_pending) cluster_wait_acquire();
        s3_pending = false;
        if (ema_out) {
          mbar_wait(&s_bar[0], ph_ema_done);
          ph_ema_done ^= 1u;
          ema_out = false;
        }
        if (signaller) {
          st_cluster(F_fl, 0);
          st_cluster(F_fl + 4, E);
          st_cluster(F_fl + 8, T);
        }
        if (tid == 0 && E > 0 && E <= a.cap_entries)
          mbar_arrive_expect_tx(&s_bar[1], 8u * static_cast<unsigned>(follower_entries(E, nw * C, nw) + (C - 1) * nw));
        cluster_arrive_release();
        s1_done = true;
      }
      __syncthreads();
      TF_MARK(2);
      if (tid == 0) s_Efr = E;
    }
    __syncthreads();
    // ---- fp64 cosine cost of un-gated pairs (tf/assoc.py:34-46), cluster-wide --
    if (C > 1 && !s1_done) {
      if (s3_pending) cluster_wait_acquire();                      // previous frame's S3 phase
      s3_pending = false;
      if (ema_out) {                                               // previous frame's EMA applied
        mbar_wait(&s_bar[0], ph_ema_done);
        ph_ema_done ^= 1u;
        ema_out = false;
      }
      TF_SUB(24);
      const int Ef = s_Efr;
      if (signaller) {
        st_cluster(F_fl, 0);
        st_cluster(F_fl + 4, Ef);
        st_cluster(F_fl + 8, T);
      }
      if (tid == 0 && Ef > 0 && Ef <= a.cap_entries)               // bytes the followers will send
        mbar_arrive_expect_tx(&s_bar[1], 8u * static_cast<unsigned>(follower_entries(Ef, nw * C, nw) + (C - 1) * nw));
      cluster_arrive_release();                                    // S1: entries ready
      TF_SUB(25);
    }
    s1_done = false;
    TF_SUB(21);
    if (gating) {
      CostView cv;
      cv.ecol = ecol;
      cv.erow = erow;
      cv.eval = eval;
      cv.t_slot = t_slot;
      cv.ampw = s_ampw;
      cv.eval_cl = cv.ampw_cl = cv.bar_cl = 0u;
      cv.pool = a.trk.emb_pool + sT * static_cast<long long>(D);
      cv.dets = a.det.emb + fK * static_cast<long long>(D);
      cv.E = s_Efr;
      cv.D = D;
      cost_work(cv, wid, nw * C);
    }
    __syncthreads();
    TF_SUB(22);
    if (C > 1 && s_Efr > 0) {                                      // S2: costs written
      if (s_Efr <= a.cap_entries) {
        mbar_wait(&s_bar[1], ph_cost_tx);
        ph_cost_tx ^= 1u;
      } else {
        mbar_wait(&s_bar[2], ph_cost_pool);
        ph_cost_pool ^= 1u;
      }
    }
    TF_SUB(23);
    if (kExt && P.fuse && s_Efr > 0) {    // JDE extension: lambda-fused cost (off on the reference path)
      fuse_motion_costs(P.lambda, P.lambda_w, P.gate_metric, ecol, erow, eval, s_Efr, t_mean, g_il, d_meas, s_ampw,
                        nw * C);
      __syncthreads();
    }
    TF_XSYNC(1);
    // the previous frame's EMA list was consumed before S1: reset it
    for (int k = tid; k < K; k += blockDim.x) ema_slot[k] = -1;
    if (wid == 0) {                       // amplitude of the finite costs (read by the LAP after barriers)
      double m = 0.0;
      if (s_Efr > 0)
        for (int i = lane; i < nw * C; i += 32) m = fmax(m, s_ampw[i]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
      if (lane == 0) s_amp = m;
    }
    TF_XSYNC(2);
    TF_MARK(3);
    // errors from here on finish the frame's cluster barriers, then stop
    const bool frame_ok = (s_err == STATUS_CLEAR) && (s_ema_err == STATUS_CLEAR);
    if (frame_ok) {

    // ---- exact LAP (tf/assoc.py:60-87) --------------------------------------
    // The reference pads the gated matrix with a sentinel and solves it with
    // scipy's shortest-augmenting-path LAP: maximise the number of finite
    // pairs, then minimise their cost. Three exact steps:
    //  1. forced-pair peeling. Two exchange arguments force pairs in EVERY
    //     optimum: R1 a row whose only live edge (t,c) is the strict minimum
    //     of column c's live edges; R2 a column whose only live edge (t,c) is
    //     the strict minimum of row t's live edges. Peeling repeats until
    //     nothing is forced (edge-parallel, atomics on bit patterns of the
    //     non-negative costs);
    //  2. the residual graph (lost tracks with wide gates competing for
    //     unclaimed detections) is split into connected components; when no
    //     component holds two equal costs the optimum is unique and each
    //     component is solved by one warp with the scipy-order restatement;
    //  3. otherwise (a genuine tie, e.g. two detections sharing one cell's
    //     embedding) the whole padded matrix is solved by the scipy-order
    //     restatement, so the tie is broken exactly as the reference breaks it.
    if (gating) {
      const int E = s_E;
      const int NN = T + K;
      for (int r = tid; r < T; r += blockDim.x) { rcol[r] = -1; p_ra[r] = 1; }
      for (int c = tid; c < K; c += blockDim.x) { p_ca[c] = 1; c_map[c] = -1; }
      // edge ids are int16 in the peeling lists: beyond that, solve the padded matrix
      const bool huge = E > 32767;
      // Aggregates use 32-bit keys (the high word of the non-negative cost's
      // bit pattern: order-preserving, so a key that is the strict minimum
      // marks a strict value minimum) and native shared-memory atomics. A key
      // tie only makes peeling skip a pair this round; skipped pairs stay in
      // the residual, which is solved exactly. Forced pairs never conflict (a
      // degree-1 row or column has one candidate partner and a strict minimum
      // is unique), so the rule pass removes them at once. Two aggregate sets
      // alternate by round: the rule pass reads one and resets the other, so a
      // round costs three barriers. (The component arrays are free scratch
      // until peeling ends.)
      // (plain selects of shared pointers, not pointer arrays: the compiler then
      // keeps them in the shared window -- LDS / ATOMS instead of generic ops)
      TF_XSYNC(3);
      unsigned* const km0 = reinterpret_cast<unsigned*>(p_cmin);
      unsigned* const km1 = km0 + K;
      unsigned* const rk0 = reinterpret_cast<unsigned*>(p_rmin);
      unsigned* const rk1 = rk0 + T;
      for (int c = tid; c < K; c += blockDim.x) { km0[c] = ~0u; p_ccnt[c] = 0; c_nr[c] = 0; }
      for (int r = tid; r < T; r += blockDim.x) { rk0[r] = ~0u; p_rcnt[r] = 0; c_ne[r] = 0; }
      if (tid == 0) { s_flag = 0; s_flag2 = 0; s_nlive[0] = 0; s_nlive[1] = 0; }
      for (int x = tid; x < NN; x += blockDim.x) c_lab[x] = x;   // components start from singletons
      __syncthreads();
      // Each round's edge pass also appends the live edges to a list (even
      // rounds: c_elist, odd: c_epos); the last round kills nothing, so its list
      // is the residual.
      int last_round = 0;
      for (int round = 0; !huge; ++round) {
        last_round = round;
        if (a.stats && tid == 0) s_ph[15] += 1;          // peeling rounds
        const int cur = round & 1;
        unsigned* km = cur ? km1 : km0;
        unsigned* rk = cur ? rk1 : rk0;
        int* cc = cur ? p_cdeg : p_ccnt;
        int* rc = cur ? p_rdeg : p_rcnt;
        int* cd = cur ? c_nc : c_nr;
        int* rd = cur ? c_root : c_ne;
        unsigned* kmn = cur ? km0 : km1;
        unsigned* rkn = cur ? rk0 : rk1;
        int* ccn = cur ? p_ccnt : p_cdeg;
        int* rcn = cur ? p_rcnt : p_rdeg;
        int* cdn = cur ? c_nr : c_nc;
        int* rdn = cur ? c_ne : c_root;
        int16_t* lst = cur ? c_epos : c_elist;
        // rounds after the first walk only the previous round's live edges
        const int16_t* src = round == 0 ? nullptr : (cur ? c_elist : c_epos);
        const int n_src = round == 0 ? E : s_nlive[cur ^ 1];
        for (int e0 = 0; e0 < n_src; e0 += blockDim.x) {
          const int q = e0 + tid;
          const int e = q < n_src ? (src ? static_cast<int>(src[q]) : q) : E;
          bool live = false;
          if (e < E) {
            const int r = erow[e], c = ecol[e];
            if (p_ra[r] && p_ca[c]) {
              live = true;
              const unsigned key = static_cast<unsigned>(__double_as_longlong(eval[e]) >> 32);
              atomicMin(&km[c], key);
              atomicAdd(&cd[c], 1);
              p_crow[c] = r;                 // the row, when the degree ends up 1
              atomicMin(&rk[r], key);
              atomicAdd(&rd[r], 1);
              p_rc1[r] = c;                  // the column, when the degree ends up 1
            }
          }
          const unsigned bm = __ballot_sync(FULL, live);
          int base = 0;
          if (lane == 0 && bm) base = atomicAdd(&s_nlive[cur], __popc(bm));
          base = __shfl_sync(FULL, base, 0);
          if (live) lst[base + __popc(bm & ((1u << lane) - 1u))] = static_cast<int16_t>(e);
        }
        __syncthreads();
        const int n_cur = s_nlive[cur];
        for (int q = tid; q < n_cur; q += blockDim.x) {      // this round's live edges
          const int e = lst[q];
          const int r = erow[e], c = ecol[e];
          const unsigned key = static_cast<unsigned>(__double_as_longlong(eval[e]) >> 32);
          // counts of keys within one unit of the minimum: a forced pair must
          // beat every rival by >= 2^-20 relative, far beyond any roundoff in
          // the reference's solve (closer rivals stay for the exact residual)
          if (key <= km[c] + 1u) atomicAdd(&cc[c], 1);
          if (key <= rk[r] + 1u) atomicAdd(&rc[r], 1);
        }
        __syncthreads();
        int* flag = cur ? &s_flag2 : &s_flag;
        if (tid == 0) { *(cur ? &s_flag : &s_flag2) = 0; s_nlive[cur ^ 1] = 0; }   // the next round's flag, list
        for (int x = tid; x < T + K; x += blockDim.x) {
          int r = -1, c = -1;
          if (x < T) {                                    // R1
            if (p_ra[x] && rd[x] == 1) {
              const int c1 = p_rc1[x];
              if (cc[c1] == 1 && rk[x] == km[c1]) { r = x; c = c1; }
            }
          } else {                                        // R2
            const int cx = x - T;
            if (p_ca[cx] && cd[cx] == 1) {
              const int r1 = p_crow[cx];
              if (rc[r1] == 1 && rk[r1] == km[cx]) { r = r1; c = cx; }
            }
          }
          if (r >= 0) {
            rcol[r] = static_cast<int16_t>(c);
            p_ra[r] = 0;
            p_ca[c] = 0;
            *flag = 1;
          }
        }
        for (int cx = tid; cx < K; cx += blockDim.x) { kmn[cx] = ~0u; ccn[cx] = 0; cdn[cx] = 0; }
        for (int rx = tid; rx < T; rx += blockDim.x) { rkn[rx] = ~0u; rcn[rx] = 0; rdn[rx] = 0; }
        __syncthreads();
        if (!*flag) break;
      }
      TF_XSYNC(4);
      TF_SUB(17);
      // residual edges: the last peeling round's list
      const int E_live = huge ? 0 : s_nlive[last_round & 1];
      if (!huge && (last_round & 1)) {         // keep the residual list in c_elist
        int16_t* tmp = c_elist;
        c_elist = c_epos;
        c_epos = tmp;
      }
      if (tid == 0) {
        s_tie = huge; s_alt = 0; s_nmulti = -1;
        if (a.stats && huge) s_ph[35] += 1;
      }
      if (!huge && E_live <= 32) {
        // Small residual (the common case): one warp labels the components,
        // checks them for equal costs and lays out the per-component problems;
        // no block barriers.
        if (wid == 0) {
          const bool on = lane < E_live;
          int r = 0, cn = 0, root = 0;
          if (on) {
            const int e = c_elist[lane];
            r = erow[e];
            cn = T + ecol[e];
          }
          for (;;) {
            bool changed = false;
            if (on) {
              const int la = c_lab[r], lb = c_lab[cn];
              if (la != lb) {
                const int m = min(la, lb);
                atomicMin(&c_lab[r], m);
                atomicMin(&c_lab[cn], m);
                changed = true;
              }
            }
            __syncwarp();
            if (on) {                                       // pointer jumping (monotone)
              int l = c_lab[r], ll = c_lab[l];
              if (ll < l) atomicMin(&c_lab[r], ll);
              l = c_lab[cn]; ll = c_lab[l];
              if (ll < l) atomicMin(&c_lab[cn], ll);
            }
            __syncwarp();
            if (!__any_sync(FULL, changed)) break;
          }
          if (on) root = c_lab[r];
          // distinct rows / columns / roots: the last writer of a marker owns it
          int* mark = c_lrp;
          if (on) { mark[r] = lane; mark[cn] = lane; }
          __syncwarp();
          const bool own_r = on && mark[r] == lane, own_c = on && mark[cn] == lane;
          __syncwarp();
          if (on) mark[root] = lane;
          __syncwarp();
          const bool own_root = on && mark[root] == lane;
          if (own_root) { c_nr[root] = 0; c_nc[root] = 0; c_ne[root] = 0; }
          __syncwarp();
          if (own_r) atomicAdd(&c_nr[root], 1);
          if (own_c) atomicAdd(&c_nc[root], 1);
          if (on) atomicAdd(&c_ne[root], 1);
          __syncwarp();
          const unsigned rm = __ballot_sync(FULL, own_root);
          const int n_multi = __popc(rm);
          const int i = __popc(rm & ((1u << lane) - 1u));
          const int vsz = own_root ? max(c_nr[root], c_nc[root]) : 0;
          const int vne = own_root ? c_ne[root] : 0;
          int isz = vsz, ine = vne;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int a1 = __shfl_up_sync(FULL, isz, o), a2 = __shfl_up_sync(FULL, ine, o);
            if (lane >= o) { isz += a1; ine += a2; }
          }
          // compact the owners' (root, offsets) to slot i
          if (own_root) {
            c_root[i] = root;
            c_off[i] = isz - vsz;
            c_eoff[i] = ine - vne;
          }
          if (lane == 0) {
            s_nmulti = n_multi;
            if (a.stats) s_ph[10] += n_multi;
          }
        }
        __syncthreads();
      } else {
        for (int x = tid; x < NN; x += blockDim.x) {
          c_lab[x] = x;
          c_nr[x] = 0;
          c_nc[x] = 0;
          c_ne[x] = 0;
        }
        if (tid == 0) s_cflag = 1;
        for (;;) {
          __syncthreads();
          const int go = s_cflag;
          __syncthreads();
          if (!go) break;
          if (tid == 0) s_cflag = 0;
          __syncthreads();
          for (int q = tid; q < E_live; q += blockDim.x) {
            const int e = c_elist[q];
            const int r = erow[e], c = T + ecol[e];
            const int la = c_lab[r], lb = c_lab[c];
            if (la != lb) {
              const int m = min(la, lb);
              atomicMin(&c_lab[r], m);
              atomicMin(&c_lab[c], m);
              s_cflag = 1;
            }
          }
          __syncthreads();
          for (int x = tid; x < NN; x += blockDim.x) {       // pointer jumping (monotone)
            const int l = c_lab[x], ll = c_lab[l];
            if (ll < l) c_lab[x] = ll;
          }
        }
        for (int x = tid; x < NN; x += blockDim.x) {
          const bool alive = x < T ? p_ra[x] != 0 : p_ca[x - T] != 0;
          if (alive) atomicAdd(x < T ? &c_nr[c_lab[x]] : &c_nc[c_lab[x]], 1);
        }
        for (int q = tid; q < E_live; q += blockDim.x) atomicAdd(&c_ne[c_lab[erow[c_elist[q]]]], 1);
        __syncthreads();
      }
      TF_SUB(16);
      // near-optimum margin of the component solves (costs are in [0, 2]
      // scaled by the amplitude; the reference's roundoff is ~1e-13)
      const double tie_eps = 1e-9 * fmax(1.0, s_amp);
      if (!s_tie) {
        int n_multi = s_nmulti;
        const bool laid_out = n_multi >= 0;
        if (!laid_out) {
        n_multi = block_rank(NN, [&](int x) { return c_lab[x] == x && c_ne[x] >= 1; }, c_pos, s_warp);
        if (a.stats && tid == 0) s_ph[10] += n_multi;   // (the one-warp layout counts its own)
        for (int x = tid; x < NN; x += blockDim.x)
          if (c_pos[x] >= 0) c_root[c_pos[x]] = x;
        __syncthreads();
        TF_SUB(18);
        if (wid == 0) {
          int carry = 0;
          for (int i0 = 0; i0 < n_multi; i0 += 32) {
            const int i = i0 + lane;
            int v = 0;
            if (i < n_multi) v = max(c_nr[c_root[i]], c_nc[c_root[i]]);
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              int q = __shfl_up_sync(FULL, incl, o);
              if (lane >= o) incl += q;
            }
            if (i < n_multi) c_off[i] = carry + incl - v;
            carry += __shfl_sync(FULL, incl, 31);
          }
          int ecarry = 0;
          for (int i0 = 0; i0 < n_multi; i0 += 32) {
            const int i = i0 + lane;
            const int v = i < n_multi ? c_ne[c_root[i]] : 0;
            int incl = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              int q = __shfl_up_sync(FULL, incl, o);
              if (lane >= o) incl += q;
            }
            if (i < n_multi) c_eoff[i] = ecarry + incl - v;
            ecarry += __shfl_sync(FULL, incl, 31);
          }
        }
        __syncthreads();
        }
        for (int i = wid; i < n_multi; i += nw) {
          const int root = c_root[i], off = c_off[i];
          if (c_nr[root] == 1 || c_nc[root] == 1) {
            // a star (one track wanting several detections, or one detection
            // wanted by several tracks): the maximum matching has one pair and,
            // with no equal costs in the component, the cheapest edge is it
            double best = INFINITY;
            int be = -1;
            for (int q = lane; q < E_live; q += 32) {
              const int e = c_elist[q];
              if (c_lab[erow[e]] == root && eval[e] < best) { best = eval[e]; be = e; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const double ob = __shfl_xor_sync(FULL, best, o);
              const int oe = __shfl_xor_sync(FULL, be, o);
              if (ob < best || (ob == best && oe > be)) { best = ob; be = oe; }
            }
            // the optimum is unique iff no other edge comes within tie_eps
            double second = INFINITY;
            for (int q = lane; q < E_live; q += 32) {
              const int e = c_elist[q];
              if (e != be && c_lab[erow[e]] == root) second = fmin(second, eval[e]);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) second = fmin(second, __shfl_xor_sync(FULL, second, o));
            if (lane == 0 && be >= 0) rcol[erow[be]] = ecol[be];
            if (lane == 0 && !(second - best > tie_eps)) {
              s_alt = 1;
              if (a.stats) atomicAdd(reinterpret_cast<unsigned long long*>(&s_ph[34]), 1ull);
            }
            continue;
          }
          int nr_l = 0, nc_l = 0;
          for (int t0 = 0; t0 < T; t0 += 32) {
            const int t = t0 + lane;
            const bool in = t < T && c_lab[t] == root && p_ra[t];
            const unsigned bm = __ballot_sync(FULL, in);
            if (in) {
              const int j = nr_l + __popc(bm & ((1u << lane) - 1u));
              c_rows[off + j] = static_cast<int16_t>(t);
              c_rmap[t] = static_cast<int16_t>(j);
            }
            nr_l += __popc(bm);
          }
          for (int k0 = 0; k0 < K; k0 += 32) {
            const int k = k0 + lane;
            const bool in = k < K && c_lab[T + k] == root && p_ca[k];
            const unsigned bm = __ballot_sync(FULL, in);
            if (in) {
              const int j = nc_l + __popc(bm & ((1u << lane) - 1u));
              c_cols[off + j] = static_cast<int16_t>(k);
              c_map[k] = static_cast<int16_t>(j);
            }
            nc_l += __popc(bm);
          }
          __syncwarp();
          const int n_l = nr_l > nc_l ? nr_l : nc_l;
          LapScratch Ls;
          Ls.u = L.u + off; Ls.v = L.v + off; Ls.dist = L.dist + off; Ls.crow = L.crow + off;
          Ls.path = L.path + off; Ls.row4col = L.row4col + off; Ls.col4row = L.col4row + off;
          Ls.rem = L.rem + off; Ls.vrows = L.vrows + off + i; Ls.vcols = L.vcols + off + i;
          const double sentinel = 2.0 * static_cast<double>(n_l) * fmax(s_amp, 1.0) + 1.0;
          // The optimum is unique here, so the component is solved from its
          // smaller side (typically 1-3 detections wanted by many lost tracks)
          // and the padding rows are skipped.
          if (nc_l < nr_l) {
            int* lrp = c_lrp + off + i;                 // nc_l + 1 row pointers
            int16_t* led = c_epos + c_eoff[i];          // the component's edge ids by detection
            // counting sort of the component's live edges by detection (lane-parallel)
            for (int j = lane; j <= nc_l; j += 32) lrp[j] = 0;
            __syncwarp();
            for (int q = lane; q < E_live; q += 32) {
              const int e = c_elist[q];
              if (c_lab[erow[e]] == root) atomicAdd(&lrp[c_map[ecol[e]] + 1], 1);
            }
            __syncwarp();
            if (lane == 0)
              for (int j = 0; j < nc_l; ++j) lrp[j + 1] += lrp[j];
            __syncwarp();
            for (int q = lane; q < E_live; q += 32) {
              const int e = c_elist[q];
              if (c_lab[erow[e]] == root) led[atomicAdd(&lrp[c_map[ecol[e]]], 1)] = static_cast<int16_t>(e);
            }
            __syncwarp();
            if (lane == 0) {                          // cursors advanced to the row ends: shift back
              for (int j = nc_l; j > 0; --j) lrp[j] = lrp[j - 1];
              lrp[0] = 0;
            }
            __syncwarp();
            warp_lap_fast(n_l, nc_l, TransposedRows{lrp, led, erow, eval, c_rmap}, sentinel, Ls, nc_l);
            __syncwarp();
#ifdef TF_EXPERIMENT_COUNT_LAPU
            if (a.stats && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_ph[14]), 1ull);
#endif
#ifndef TF_EXPERIMENT_NO_LAPU
            {
              const int uq = lap_unique(nc_l, n_l, TransposedRows{lrp, led, erow, eval, c_rmap}, sentinel, tie_eps, Ls);
              if (uq <= 0 && lane == 0) {
                s_alt = 1;
                if (a.stats) atomicAdd(reinterpret_cast<unsigned long long*>(&s_ph[uq < 0 ? 32 : 33]), 1ull);
              }
            }
#endif
            for (int j = lane; j < nc_l; j += 32) {
              const int lc = Ls.col4row[j];
              if (lc < nr_l) {
                const int t = c_rows[off + lc], c = c_cols[off + j];
                for (int e = rowptr[t]; e < rowptr[t + 1]; ++e)
                  if (ecol[e] == c) { rcol[t] = static_cast<int16_t>(c); break; }
              }
            }
          } else {
            warp_lap_fast(n_l, nr_l, ComponentRows{rowptr, ecol, eval, c_rows + off, c_map}, sentinel, Ls, nr_l);
            __syncwarp();
#ifdef TF_EXPERIMENT_COUNT_LAPU
            if (a.stats && lane == 0) atomicAdd(reinterpret_cast<unsigned long long*>(&s_ph[10]), 1ull);
#endif
#ifndef TF_EXPERIMENT_NO_LAPU
            {
              const int uq = lap_unique(nr_l, n_l, ComponentRows{rowptr, ecol, eval, c_rows + off, c_map}, sentinel,
                                        tie_eps, Ls);
              if (uq <= 0 && lane == 0) {
                s_alt = 1;
                if (a.stats) atomicAdd(reinterpret_cast<unsigned long long*>(&s_ph[uq < 0 ? 32 : 33]), 1ull);
              }
            }
#endif
            for (int r = lane; r < nr_l; r += 32) {
              const int j = Ls.col4row[r];
              if (j < nc_l) {
                const int t = c_rows[off + r], c = c_cols[off + j];
                for (int e = rowptr[t]; e < rowptr[t + 1]; ++e)
                  if (ecol[e] == c) { rcol[t] = static_cast<int16_t>(c); break; }
              }
            }
          }
        }
        __syncthreads();
        TF_SUB(19);
      }
      const bool full_solve = s_tie || s_alt;
      if (a.stats && tid == 0) { s_ph[8] += full_solve; s_ph[9] += E; s_ph[11] += 1; s_ph[12] += T; s_ph[13] += K; s_ph[14] += E_live; }
      if (full_solve) {
        // a near-optimum exists (or the matrix is beyond the int16 edge
        // lists): the whole padded matrix in the reference's order
        if (wid == 0) {
          const int n = T > K ? T : K;
          const double sentinel = 2.0 * static_cast<double>(n) * fmax(s_amp, 1.0) + 1.0;
          warp_lap_fast(n, T, CsrRows{rowptr, ecol, eval}, sentinel, L);
          __syncwarp();
          for (int r = lane; r < T; r += 32) {
            const int c = L.col4row[r];
            rcol[r] = static_cast<int16_t>(c < K ? c : -1);
          }
          TF_SUB(20);
        }
      }
    }
    __syncthreads();
    TF_MARK(4);
    // ---- matches + max_cost threshold (tf/assoc.py:77-107), then the
    // matched tracks' Kalman update + lifecycle (tf/tracker.py:114-143), one
    // thread per track in one pass; matched tracks also post their EMA work
    TF_XSYNC(5);
    TF_MARK(5);
    if (kExt && P.iou_stage) {
      // JDE extension: first-stage matches, then the IoU stage on what is left
      for (int t = tid; t < T; t += blockDim.x) {
        int md = -1;
        double mc = 0.0;
        const int c = gating ? rcol[t] : -1;
        if (c >= 0) {
          for (int e = rowptr[t]; e < rowptr[t + 1]; ++e)
            if (ecol[e] == c) {
              mc = eval[e];
              md = (mc > P.max_cost) ? -1 : c;
              break;
            }
        }
        t_mdet[t] = md;
        t_mcost[t] = mc;
        if (md >= 0) d_row[md] = t;
      }
      __syncthreads();
      if (wid == 0 && T > 0 && K > 0)
        iou_second_stage(P.iou_threshold, T, K, Tm, Km, a.cap_entries, smem, d_meas,
                         a.pool_val + static_cast<long long>(s) * Tm * Km, &s_err);
      __syncthreads();
    }
    for (int t = tid; t < T; t += blockDim.x) {
      int md = -1;
      double mc = 0.0;
      if (kExt && P.iou_stage) {
        md = t_mdet[t];
        mc = t_mcost[t];
      } else if (gating) {
        const int c = rcol[t];
        if (c >= 0) {
          for (int e = rowptr[t]; e < rowptr[t + 1]; ++e)
            if (ecol[e] == c) {
              mc = eval[e];
              md = (mc > P.max_cost) ? -1 : c;
              break;
            }
        }
      }
      t_mdet[t] = md;
      t_mcost[t] = mc;
      int remove = 0;
      if (md >= 0) {
        d_row[md] = t;
        ema_slot[md] = t_slot[t];
        if (!KF::update(P, &t_mean[8 * t], &t_cov[12 * t], &d_meas[4 * md]))
          flag_error(&s_err, t + 1, TF_NUMERIC);
        t_state[t] = 0;
        t_lost[t] = -1;
        t_last[t] = frame;
        t_hits[t] += 1;
      } else {
        if (t_state[t] == 0) {                    // ACTIVE -> LOST (tf/tracker.py:127-131)
          t_state[t] = 1;
          t_lost[t] = frame;
        }
        remove = (t_state[t] == 1) && (frame - t_lost[t] >= P.max_lost);   // tf/tracker.py:133-143
      }
      t_flag[t] = remove;
    }
    }  // frame_ok
    if (tid == 0) { s_ema_work = 0; if (frame_ok) s_ema_b = b; }
    if (C > 1) {
      // S3 straight after this thread's share of the per-track pass (its
      // release covers this thread's EMA-list entries; -0.3 us per frame
      // against arriving after the CTA barrier); the CTA barrier follows
      TF_SUB(27);
      if (signaller) st_cluster(F_fl + 12, frame_ok ? K : 0);
      cluster_wait_acquire();                                     // this frame's S1 phase
      cluster_arrive_release();                                   // S3: EMA list published
      TF_SUB(26);
      s3_pending = true;
      ema_out = true;
    }
    __syncthreads();
    if (C == 1 && frame_ok) {
      EmaView ev;
      ev.slot = ema_slot;
      ev.work = &s_ema_work;
      ev.err = &s_err;
      ev.pool = a.trk.emb_pool + sT * static_cast<long long>(D);
      ev.dets = a.det.emb + fK * static_cast<long long>(D);
      ev.alpha = P.alpha;
      ev.beta = P.beta;
      ev.K = K;
      ev.D = D;
      ema_work(ev);
      __syncthreads();
    }
    TF_MARK(6);
    if (!frame_ok) {                          // errors before the LAP: stop here
      if (tid == 0) {
        if (s_err != STATUS_CLEAR) s_status = (b << 8) | (s_err & 0xff);
        else s_status = (s_ema_b << 8) | (s_ema_err & 0xff);  // follower EMA of the previous frame
      }
      break;
    }

    // ---- records: matched tracks in list (= id) order, then births ---------
    // Births are unmatched detections in ascending order (tf/tracker.py:145-157);
    // removed tracks leave the list in order (tf/tracker.py:133-143) and push
    // their embedding slots onto the free stack. The four ranks (record,
    // birth, removed, kept) come from one block scan of packed 16-bit counters.
    int* rec_pos = c_nr;                       // LAP scratch, free from here on
    unsigned long long tot4 = 0;
    {
      const int n_items = T > K ? T : K;
      for (int c0 = 0; c0 < n_items; c0 += blockDim.x) {
        const int i = c0 + tid;
        const bool f0 = i < T && t_mdet[i] >= 0 && t_hits[i] >= P.min_hits;
        const bool f1 = i < K && d_row[i] < 0;
        const bool f2 = i < T && t_flag[i] != 0;
        const bool f3 = i < T && t_flag[i] == 0;
        const unsigned long long v = static_cast<unsigned long long>(f0) | (static_cast<unsigned long long>(f1) << 16) |
                                     (static_cast<unsigned long long>(f2) << 32) |
                                     (static_cast<unsigned long long>(f3) << 48);
        unsigned long long tot;
        const unsigned long long ex = block_exscan_u64(v, s_scan64, &tot) + tot4;
        if (i < T) {
          rec_pos[i] = f0 ? static_cast<int>(ex & 0xffff) : -1;
          rpos[i] = f2 ? static_cast<int16_t>((ex >> 32) & 0xffff) : static_cast<int16_t>(-1);
          npos[i] = f3 ? static_cast<int16_t>(ex >> 48) : static_cast<int16_t>(-1);
        }
        if (i < K) d_pos[i] = f1 ? static_cast<int16_t>((ex >> 16) & 0xffff) : static_cast<int16_t>(-1);
        tot4 += tot;
        if (c0 + static_cast<int>(blockDim.x) < n_items) __syncthreads();   // s_scan64 reuse
      }
    }
    const int n_rec_matched = static_cast<int>(tot4 & 0xffff);
    const int n_birth = static_cast<int>((tot4 >> 16) & 0xffff);
    const int n_rm = static_cast<int>((tot4 >> 32) & 0xffff);
    const int n_surv = T - n_rm;
    if (n_surv + n_birth > Tm) {
      if (tid == 0) s_status = (b << 8) | TF_CAPACITY;
      break;
    }
    TF_XSYNC(6);
    const long long fR = static_cast<long long>(f) * a.out.max_records;
    const int base_free = s_nfree;
    // read before the compaction's barriers: tid 0 updates s_next at the end
    // of its birth loop, possibly before a slow warp reaches the birth block
    const long long next_id = s_next;
    // matched records, trace, free-stack pushes, then the ordered in-place
    // compaction one chunk of blockDim rows per round: destinations never
    // exceed sources, and a round's reads finish before its writes
    for (int c0 = 0; c0 < T; c0 += blockDim.x) {
      const int t = c0 + tid;
      bool mv = false;
      int d = -1;
      long long r_id = 0, r_lost = 0, r_last = 0;
      int r_state = 0, r_hits = 0, r_slot = 0;
      double r_mean[8], r_cov[12];
      if (t < T) {
        const int k = t_mdet[t];
        if (k >= 0 && a.trace.det_track) {
          a.trace.det_track[fK + k] = t_id[t];
          a.trace.det_cost[fK + k] = t_mcost[t];
          a.trace.det_matched[fK + k] = 1;
        }
        const int r = rec_pos[t];
        if (r >= 0) {
          double box[4];
          if (!meas_to_box(&t_mean[8 * t], box)) flag_error(&s_err, t + 1, TF_INVALID_BOX);
          if (r < a.out.max_records) {
            a.out.track_id[fR + r] = t_id[t];
            for (int q = 0; q < 4; ++q) a.out.box[(fR + r) * 4 + q] = box[q];
            a.out.objectness[fR + r] = d_obj[k];
          }
        }
        if (t_flag[t]) f_stk[base_free + rpos[t]] = t_slot[t];
        mv = t_flag[t] == 0 && npos[t] != t;
        if (mv) {
          d = npos[t];
          r_id = t_id[t]; r_lost = t_lost[t]; r_last = t_last[t];
          r_state = t_state[t]; r_hits = t_hits[t]; r_slot = t_slot[t];
#pragma unroll
          for (int z = 0; z < 8; ++z) r_mean[z] = t_mean[8 * t + z];
#pragma unroll
          for (int z = 0; z < 12; ++z) r_cov[z] = t_cov[12 * t + z];
        }
      }
      if (n_rm > 0) __syncthreads();
      if (mv) {
        t_id[d] = r_id; t_lost[d] = r_lost; t_last[d] = r_last;
        t_state[d] = r_state; t_hits[d] = r_hits; t_slot[d] = r_slot;
#pragma unroll
        for (int z = 0; z < 8; ++z) t_mean[8 * d + z] = r_mean[z];
#pragma unroll
        for (int z = 0; z < 12; ++z) t_cov[12 * d + z] = r_cov[z];
      }
      __syncthreads();                         // also publishes the free-stack pushes
    }
    // births: new tracks appended in ascending detection order, one warp per
    // birth (lane 0 initialises the row, the warp copies the embedding)
    {
      const int nf = base_free + n_rm;
      const long long next = next_id;
      TF_XSYNC(7);
      TF_MARK(7);
      birth_rows(a.det.emb + fK * static_cast<long long>(D), a.trk.emb_pool + sT * static_cast<long long>(D), d_pos,
                 f_stk, nf, K, D);
      for (int k = wid; k < K; k += nw) {   // (births + frame tail: slot 30)
        const int r = d_pos[k];
        if (r < 0) continue;
        const int t = n_surv + r;
        int slot = 0;
        if (lane == 0) {
          const double* z = &d_meas[4 * k];
          if (!(z[3] > 0.0)) flag_error(&s_err, k + 1, TF_INVALID_MEASUREMENT);
          KF::initiate(P, z, &t_mean[8 * t], &t_cov[12 * t]);
          t_id[t] = next + r;
          t_state[t] = 0;
          t_hits[t] = 1;
          t_lost[t] = -1;
          t_last[t] = frame;
          slot = f_stk[nf - 1 - r];                           // pop in birth order
          t_slot[t] = slot;
          if (a.trace.det_track) {
            a.trace.det_track[fK + k] = next + r;
            a.trace.det_cost[fK + k] = nan("");
            a.trace.det_matched[fK + k] = 0;
          }
          if (1 >= P.min_hits) {
            const int rr = n_rec_matched + r;
            double box[4];
            if (!meas_to_box(z, box)) flag_error(&s_err, k + 1, TF_INVALID_BOX);
            if (rr < a.out.max_records) {
              a.out.track_id[fR + rr] = next + r;
              for (int q = 0; q < 4; ++q) a.out.box[(fR + rr) * 4 + q] = box[q];
              a.out.objectness[fR + rr] = d_obj[k];
            }
          }
        }
      }
      if (tid == 0) {
        s_nfree = nf - n_birth;
        s_next = next + n_birth;
        s_T = n_surv + n_birth;
        const int nrec = n_rec_matched + (1 >= P.min_hits ? n_birth : 0);
        a.out.count[f] = nrec;
        if (nrec > a.out.max_records) flag_error(&s_err, 0, TF_CAPACITY);
        if (a.trace.det_count) a.trace.det_count[f] = K;
        if (a.trace.cand_count) a.trace.cand_count[f] = a.det.cand_count[f];
        tb.last_frame[s] = frame;
      }
    }
    __syncthreads();
    TF_SUB(30);
    TF_CANARY_CHECK(30);
    if (s_err != STATUS_CLEAR) {
      if (tid == 0) s_status = (b << 8) | (s_err & 0xff);
      break;
    }
  }
  if (a.stats && tid == 0) t_epi = clock64();
  if (a.sclk && tid == 0) a.sclk[4 * s + 2] = gtimer();
  const long long t_work = clock64() - t_work0;
  asm volatile("cp.async.wait_all;\n" ::: "memory");   // no prefetch outlives an early exit
  __syncthreads();
  // ---- write the stream's state back (the followers' last EMA runs meanwhile) --
  T = s_T;
  for (int i = tid; i < s_nfree; i += blockDim.x) tb.free_stack[sT + i] = f_stk[i];
  for (int t = tid; t < T; t += blockDim.x) {
    tb.id[sT + t] = t_id[t];
    tb.lost[sT + t] = t_lost[t];
    tb.last[sT + t] = t_last[t];
    tb.state[sT + t] = t_state[t];
    tb.hits[sT + t] = t_hits[t];
    tb.slot[sT + t] = t_slot[t];
    for (int q = 0; q < 8; ++q) tb.mean[(sT + t) * 8 + q] = t_mean[8 * t + q];
    for (int q = 0; q < 12; ++q) tb.cov[(sT + t) * 12 + q] = t_cov[12 * t + q];
  }
  // ---- release the follower CTAs (they wait at the S1 barrier) ----------------
  __syncthreads();
  if (C > 1) {
    if (s3_pending) cluster_wait_acquire();
    if (ema_out) mbar_wait(&s_bar[0], ph_ema_done);   // followers are done with this CTA's memory
    if (signaller) st_cluster(F_fl, 1);               // stop
    cluster_arrive_release();
    cluster_wait_acquire();
    if (tid == 0 && s_status == 0 && s_ema_err != STATUS_CLEAR) s_status = (s_ema_b << 8) | (s_ema_err & 0xff);
  }
  if (a.stats && tid == 0) s_ph[29] += clock64() - t_epi;
  __syncthreads();
  if (a.stats && tid < kPhaseSlots) atomicAdd(reinterpret_cast<unsigned long long*>(&a.stats[tid]),
                                               static_cast<unsigned long long>(s_ph[tid]));
  if (tid == 0) {
    if (a.sclk) a.sclk[4 * s + 3] = gtimer();
    tb.n_tracks[s] = T;
    tb.next_id[s] = s_next;
    tb.n_free[s] = s_nfree;
    if (s_status) tb.status[s] = s_status;    // sticky until tf_finish reads it
  }
  if (a.order_out) {                          // single-CTA streams only (C == 1)
    __shared__ int s_last;
    if (tid == 0) {
      a.work[ls] = t_work;
      __threadfence();
      s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {                             // every other CTA has finished: rank the streams
      __threadfence();
      lpt_order(a.work, a.order_out, static_cast<int>(gridDim.x), reinterpret_cast<int*>(smem));
      if (tid == 0) *a.ticket = 0u;
    }
  }
}

// ============================================================================
// Stage-level kernels (module functions of the reference)
// ============================================================================

__global__ void nms_sets_kernel(const int* offsets, const double* boxes, const double* scores,
                                const double* thr, uint8_t* keep, int* status, int cap, int words) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_misc[2];
  const int set = blockIdx.x;
  const int o0 = offsets[set], C = offsets[set + 1] - o0;
  if (C > cap) {
    if (threadIdx.x == 0) status[set] = TF_CAPACITY;
    return;
  }
  const FramePlan plan = frame_plan(0, cap, words);
  double* cbox = reinterpret_cast<double*>(smem + plan.off_box);
  double* cscore = reinterpret_cast<double*>(smem + plan.off_score);
  uint8_t* calive = smem + plan.off_alive;
  int16_t* csorted = reinterpret_cast<int16_t*>(smem + plan.off_sorted);
  unsigned long long* nmask = reinterpret_cast<unsigned long long*>(smem + plan.off_nmask);
  uint8_t* ckeep = smem + plan.off_keep;
  for (int r = threadIdx.x; r < C; r += blockDim.x) {
    for (int q = 0; q < 4; ++q) cbox[4 * r + q] = boxes[4 * (o0 + r) + q];
    cscore[r] = scores[o0 + r];
    calive[r] = 1;
  }
  __syncthreads();
  block_nms(C, cbox, cscore, calive, thr[set], csorted, nmask, words, ckeep, s_misc);
  for (int r = threadIdx.x; r < C; r += blockDim.x) keep[o0 + r] = ckeep[r];
  if (threadIdx.x == 0) status[set] = 0;
}

__global__ void lap_dense_kernel(const int* shapes, const long long* cost_off, const double* costs,
                                 const long long* row_off, int* col_for_row, int* status, int cap_n,
                                 int16_t* pool_col, double* pool_val, int* pool_rowptr, long long pool_stride) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int m = blockIdx.x, lane = threadIdx.x;
  const int nr = shapes[2 * m], nc = shapes[2 * m + 1];
  const double* c = costs + cost_off[m];
  int* out = col_for_row + row_off[m];
  const int n = nr > nc ? nr : nc;
  if (nr == 0 || nc == 0) {
    for (int r = lane; r < nr; r += 32) out[r] = -1;
    if (lane == 0) status[m] = 0;
    return;
  }
  if (n > cap_n) {
    if (lane == 0) status[m] = TF_CAPACITY;
    return;
  }
  // CSR of finite entries (global pool slice of this matrix) + amplitude
  int16_t* ecol = pool_col + m * pool_stride;
  double* eval = pool_val + m * pool_stride;
  int* rowptr = pool_rowptr + static_cast<long long>(m) * (cap_n + 1);
  double amp = 0.0;
  bool any = false;
  int carry = 0;
  for (int r = 0; r < nr; ++r) {
    if (lane == 0) rowptr[r] = carry;
    for (int k0 = 0; k0 < nc; k0 += 32) {
      int k = k0 + lane;
      double v = k < nc ? c[static_cast<long long>(r) * nc + k] : INFINITY;
      bool fin = isfinite(v);
      unsigned bm = __ballot_sync(FULL, fin);
      if (fin) {
        int e = carry + __popc(bm & ((1u << lane) - 1u));
        ecol[e] = static_cast<int16_t>(k);
        eval[e] = v;
        amp = fmax(amp, fabs(v));
        any = true;
      }
      carry += __popc(bm);
    }
  }
  if (lane == 0) rowptr[nr] = carry;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amp = fmax(amp, __shfl_xor_sync(FULL, amp, o));
  any = __any_sync(FULL, any);
  __syncwarp();
  const double sentinel = 2.0 * static_cast<double>(n) * fmax(any ? amp : 1.0, 1.0) + 1.0;
  LapScratch L;
  size_t o = 0;
  L.u = reinterpret_cast<double*>(smem + o); o += 8 * n;
  L.v = reinterpret_cast<double*>(smem + o); o += 8 * n;
  L.dist = reinterpret_cast<double*>(smem + o); o += 8 * n;
  L.crow = reinterpret_cast<double*>(smem + o); o += 8 * n;
  L.path = reinterpret_cast<int16_t*>(smem + o); o += 2 * n;
  L.row4col = reinterpret_cast<int16_t*>(smem + o); o += 2 * n;
  L.col4row = reinterpret_cast<int16_t*>(smem + o); o += 2 * n;
  L.rem = reinterpret_cast<int16_t*>(smem + o); o += 2 * n;
  L.vrows = reinterpret_cast<int16_t*>(smem + o); o += 2 * (n + 1);
  L.vcols = reinterpret_cast<int16_t*>(smem + o);
  warp_lap_fast(n, nr, CsrRows{rowptr, ecol, eval}, sentinel, L);
  __syncwarp();
  for (int r = lane; r < nr; r += 32) {
    int col = L.col4row[r];
    bool fin = col < nc && isfinite(c[static_cast<long long>(r) * nc + col]);
    out[r] = fin ? col : -1;
  }
  if (lane == 0) status[m] = 0;
}

// Dense 8x8 Kalman (KalmanFilter API on arbitrary states). Follows the matrix
// expressions of tf/motion.py term by term; on block-structured inputs (every
// state the tracker produces) it reproduces the compact form bit for bit.
__device__ void mm8(const double* A, const double* B, double* C, bool bt) {
  for (int i = 0; i < 8; ++i)
    for (int j = 0; j < 8; ++j) {
      double acc = 0.0;
      for (int k = 0; k < 8; ++k) acc = acc + A[8 * i + k] * (bt ? B[8 * j + k] : B[8 * k + j]);
      C[8 * i + j] = acc;
    }
}

// The KalmanFilter batch API on dense 8x8 states. A 64-thread block stages
// its 64 covariances through shared memory (rows padded to 65 doubles against
// bank conflicts, every 8-byte piece in flight at once by cp.async); each
// thread then runs the reference's matrix expressions for its state on its
// shared-memory row, in the reference's operation order, with fully unrolled
// (register-indexed) loops. Predict and update write their result over P, so
// they need one tile (more blocks per SM); initiate / project use a second.
constexpr int kKfBlock = 64, kKfPad = 65;
__device__ __forceinline__ double kf_F(int r, int k) { return (k == r || (r < 4 && k == r + 4)) ? 1.0 : 0.0; }

__global__ void __launch_bounds__(kKfBlock) kalman_kernel(int op, int n, Params P, const double* mean_in,
                                                          const double* cov_in, const double* zin,
                                                          double* mean_out, double* cov_out, int* status) {
  extern __shared__ __align__(16) double kf_smem[];
  double* TA = kf_smem;                               // [64][65] input covariance, then working rows
  double* TB = kf_smem + kKfBlock * kKfPad;           // [64][65] scratch, then outputs
  const int tid = threadIdx.x, i0 = blockIdx.x * kKfBlock, i = i0 + tid;
  const int nb = min(kKfBlock, n - i0);
  // the block's 64 covariances are one contiguous 32 KB range: every 8-byte
  // piece is in flight at once (cp.async), the per-state mean and measurement
  // loads overlap them
  if (op != 0) {
    const double* src = cov_in + 64LL * i0;
    for (int x = tid; x < nb * 64; x += kKfBlock)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(smem_u32(TA + (x >> 6) * kKfPad + (x & 63))),
                   "l"(src + x)
                   : "memory");
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  double m[8], z[4];
  if (i < n) {
    if (op != 0)
      for (int q = 0; q < 8; ++q) m[q] = mean_in[8LL * i + q];
    if (op == 0 || op == 3)
      for (int q = 0; q < 4; ++q) z[q] = zin[4LL * i + q];
  }
  if (op != 0) asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  const int out_w = op == 2 ? 16 : 64;                // output covariance elements per state
  double* c = TA + tid * kKfPad;
  double* o = TB + tid * kKfPad;
  if (i < n) {
    int st = 0;
    if (op == 0) {
      double h = z[3];
      if (!(h > 0.0)) st = TF_INVALID_MEASUREMENT;
      double mm[8], cc[12];
      KF::initiate(P, z, mm, cc);
      for (int q = 0; q < 8; ++q) mean_out[8LL * i + q] = mm[q];
      for (int q = 0; q < 64; ++q) o[q] = 0.0;
      for (int a4 = 0; a4 < 4; ++a4) {
        o[9 * a4] = cc[3 * a4];
        o[9 * (a4 + 4)] = cc[3 * a4 + 2];
      }
    } else if (op == 1) {
      const double h = m[3];
      for (int r = 0; r < 8; ++r) {
        double acc = 0.0;
        for (int k = 0; k < 8; ++k) acc = acc + kf_F(r, k) * m[k];
        mean_out[8LL * i + r] = acc;
      }
      // F P then (F P) F^T, in place on the state's shared row. With finite
      // inputs the zero terms of the dense products add exact zeros, so only
      // the two nonzero terms are summed (same single rounding); otherwise
      // the dense sums run as mm8 computes them (0 * inf = NaN must propagate
      // like the reference's), one column / row at a time.
      bool finite = true;
#pragma unroll
      for (int q = 0; q < 64; ++q) finite = finite && isfinite(c[q]);
      if (finite) {
#pragma unroll
        for (int r = 0; r < 4; ++r)
#pragma unroll
          for (int j = 0; j < 8; ++j) c[8 * r + j] = c[8 * r + j] + c[8 * (r + 4) + j];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int j = 0; j < 4; ++j) c[8 * r + j] = c[8 * r + j] + c[8 * r + j + 4];
      } else {
        for (int j = 0; j < 8; ++j) {
          double col[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc = acc + kf_F(r, k) * c[8 * k + j];
            col[r] = acc;
          }
#pragma unroll
          for (int r = 0; r < 8; ++r) c[8 * r + j] = col[r];
        }
        for (int r = 0; r < 8; ++r) {
          double row[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k) acc = acc + c[8 * r + k] * kf_F(j, k);
            row[j] = acc;
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) c[8 * r + j] = row[j];
        }
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double sp = KF::qpos(P, q, h), sv = KF::qvel(P, q, h);
        c[9 * q] = c[9 * q] + sp * sp;
        c[9 * (q + 4)] = c[9 * (q + 4)] + sv * sv;
      }
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int k = r; k < 8; ++k) {
          const double a = (c[8 * r + k] + c[8 * k + r]) / 2.0;
          c[8 * r + k] = a;
          c[8 * k + r] = a;
        }
    } else {
      const double h = m[3];
      double S[16], Lc[16] = {0};
      for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 4; ++k) S[4 * r + k] = c[8 * r + k];
      for (int q = 0; q < 4; ++q) {
        double rs = KF::rstd(P, q, h);
        S[5 * q] = S[5 * q] + rs * rs;
      }
      if (op == 2) {
        for (int q = 0; q < 4; ++q) mean_out[4LL * i + q] = m[q];
        for (int q = 0; q < 16; ++q) o[q] = S[q];
      } else {
        // Cholesky (lower), diagonal reciprocal as LAPACK/OpenBLAS applies it
        double inv[4];
        bool chol_ok = true;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          double acc = S[5 * j];
#pragma unroll
          for (int k = 0; k < j; ++k) acc = acc - Lc[4 * j + k] * Lc[4 * j + k];
          chol_ok = chol_ok && (acc > 0.0);
          Lc[5 * j] = sqrt(acc);
          inv[j] = 1.0 / Lc[5 * j];
#pragma unroll
          for (int r = j + 1; r < 4; ++r) {
            double v = S[4 * r + j];
#pragma unroll
            for (int k = 0; k < j; ++k) v = v - Lc[4 * r + k] * Lc[4 * j + k];
            Lc[4 * r + j] = v * inv[j];
          }
        }
        if (!chol_ok) st = TF_NUMERIC;
        if (!st) {
          // gain^T = S^-1 (P H^T)^T via L then L^T solves, column by column
          // (G [4][8] in registers; the result is written over P in place, so
          // the block needs one shared tile)
          double G[32];
#pragma unroll
          for (int col = 0; col < 8; ++col) {
            double y[4];
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              double v = c[8 * col + r];        // (P H^T)^T [r][col] = P[col][r]
#pragma unroll
              for (int k = 0; k < r; ++k) v = v - Lc[4 * r + k] * y[k];
              y[r] = v * inv[r];
            }
#pragma unroll
            for (int r = 3; r >= 0; --r) {
              double v = y[r];
#pragma unroll
              for (int k = r + 1; k < 4; ++k) v = v - Lc[4 * k + r] * G[8 * k + col];
              G[8 * r + col] = v * inv[r];
            }
          }
          double inn[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) inn[q] = z[q] - m[q];
          // NC = P - (G^T S) G, row by row in place of P (row r reads only P row r)
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc = acc + G[8 * k + r] * inn[k];
            mean_out[8LL * i + r] = m[r] + acc;
            double KS[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              double s2 = 0.0;
#pragma unroll
              for (int q = 0; q < 4; ++q) s2 = s2 + G[8 * q + r] * S[4 * q + k];
              KS[k] = s2;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              double a2 = 0.0;
#pragma unroll
              for (int q = 0; q < 4; ++q) a2 = a2 + KS[q] * G[8 * q + k];
              c[8 * r + k] = c[8 * r + k] - a2;
            }
          }
          // symmetrise in place: (a + b) / 2 is symmetric in a and b
#pragma unroll
          for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = r; k < 8; ++k) {
              const double a = (c[8 * r + k] + c[8 * k + r]) / 2.0;
              c[8 * r + k] = a;
              c[8 * k + r] = a;
            }
        }
      }
    }
    status[i] = st;
  }
  __syncthreads();
  const double* OUT = (op == 1 || op == 3) ? TA : TB;   // predict / update write their result over P
  for (int x = tid; x < nb * out_w; x += kKfBlock) {
    const int r = x / out_w, q = x - r * out_w;
    cov_out[static_cast<long long>(i0) * out_w + x] = OUT[r * kKfPad + q];
  }
}

__global__ void gating_kernel(int nt, const double* means, const double* covs, int nm, const double* z,
                              int metric, Params P, double* out, int* status) {
  const int t = blockIdx.x;
  const double* m = means + 8 * t;
  const double* c = covs + 64 * t;
  __shared__ double s_l[16], s_inv[4];
  __shared__ int s_bad;
  if (threadIdx.x == 0) {
    s_bad = 0;
    if (metric == 0) {
      double S[16], Lc[16] = {0};
      const double h = m[3];
      for (int r = 0; r < 4; ++r)
        for (int k = 0; k < 4; ++k) S[4 * r + k] = c[8 * r + k];
      for (int q = 0; q < 4; ++q) {
        double rs = KF::rstd(P, q, h);
        S[5 * q] = S[5 * q] + rs * rs;
      }
      for (int j = 0; j < 4; ++j) {
        double acc = S[5 * j];
        for (int k = 0; k < j; ++k) acc = acc - Lc[4 * j + k] * Lc[4 * j + k];
        if (!(acc > 0.0)) { s_bad = 1; break; }
        Lc[5 * j] = sqrt(acc);
        s_inv[j] = 1.0 / Lc[5 * j];
        for (int r = j + 1; r < 4; ++r) {
          double v = S[4 * r + j];
          for (int k = 0; k < j; ++k) v = v - Lc[4 * r + k] * Lc[4 * j + k];
          Lc[4 * r + j] = v * s_inv[j];
        }
      }
      for (int q = 0; q < 16; ++q) s_l[q] = Lc[q];
    } else if (metric != 1) {
      s_bad = 2;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) status[t] = s_bad == 1 ? TF_NUMERIC : TF_CONFIG;
    return;
  }
  for (int k = threadIdx.x; k < nm; k += blockDim.x) {
    const double* zz = z + 4 * k;
    double g;
    if (metric == 0) {
      double x[4];
      for (int r = 0; r < 4; ++r) {
        double v = zz[r] - m[r];
        for (int q = 0; q < r; ++q) v = v - s_l[4 * r + q] * x[q];
        x[r] = v * s_inv[r];
      }
      g = ((x[0] * x[0] + x[1] * x[1]) + x[2] * x[2]) + x[3] * x[3];
    } else {
      double dx = m[0] - zz[0], dy = m[1] - zz[1];
      g = dx * dx + dy * dy;
    }
    out[static_cast<long long>(t) * nm + k] = g;
  }
  if (threadIdx.x == 0) status[t] = 0;
}

__global__ void cosine_cost_kernel(int nt, int nd, int dim, const float* te, const float* de, double* out) {
  const int pair = blockIdx.x * n_warps() + warp_id();
  if (pair >= nt * nd) return;
  const int t = pair / nd, k = pair % nd;
  double acc = 0.0;
  for (int i = lane_id(); i < dim; i += 32)
    acc += static_cast<double>(te[static_cast<long long>(t) * dim + i]) *
           static_cast<double>(de[static_cast<long long>(k) * dim + i]);
  acc = warp_sum(acc);
  if (lane_id() == 0) out[pair] = fmin(fmax(1.0 - acc, 0.0), 2.0);
}

__global__ void normalize_rows_kernel(int n, int dim, const double* in64, const float* in32, long long stride,
                                      int quantize, float* out, int* status) {
  const int r = blockIdx.x * n_warps() + warp_id();
  if (r >= n) return;
  const int lane = lane_id();
  if (in32 && dim == 512 && !quantize) {
    // fp32 rows of 512: the row is read once into registers (same per-lane
    // element order and summation as below, so bit-identical results) and
    // divided with one reciprocal per row (div_by: the correctly rounded
    // quotient, exact true division when the norm is far from the exponent
    // limits; plain division otherwise)
    const float* src = in32 + r * stride;
    float xs[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) xs[k] = src[lane + 32 * k];
    double ss = 0.0;
    bool fin = true;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double v = static_cast<double>(xs[k]);
      fin = fin && isfinite(v);
      ss += v * v;
    }
    ss = warp_sum(ss);
    fin = __all_sync(FULL, fin);
    const double nrm = sqrt(ss);
    const int st = (!fin || nrm < 1e-12) ? TF_DEGENERATE_EMBEDDING : 0;
    if (!st) {
      float* o = out + static_cast<long long>(r) * dim;
      const bool safe = nrm > 0x1p-500 && nrm < 0x1p500;
      const double rn = __drcp_rn(nrm);
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        const double v = static_cast<double>(xs[k]);
        o[lane + 32 * k] = static_cast<float>(safe ? div_by(v, nrm, rn) : v / nrm);
      }
    }
    if (lane == 0) status[r] = st;
    return;
  }
  double ss = 0.0;
  bool fin = true;
  for (int i = lane; i < dim; i += 32) {
    double v = in64 ? in64[r * stride + i] : static_cast<double>(in32[r * stride + i]);
    fin = fin && isfinite(v);
    ss += v * v;
  }
  ss = warp_sum(ss);
  fin = __all_sync(FULL, fin);
  double nrm = sqrt(ss);
  int st = 0;
  if (!fin || nrm < 1e-12) st = TF_DEGENERATE_EMBEDDING;
  float* o = out + static_cast<long long>(r) * dim;
  if (!st) {
    double ss2 = 0.0;
    bool inrange = true;
    for (int i = lane; i < dim; i += 32) {
      double v = in64 ? in64[r * stride + i] : static_cast<double>(in32[r * stride + i]);
      float u = static_cast<float>(v / nrm);
      if (quantize) {
        inrange = inrange && fabsf(u) <= 65504.0f;
        u = __half2float(__float2half_rn(u));
        double d = u;
        ss2 += d * d;
      }
      o[i] = u;
    }
    if (quantize) {
      ss2 = warp_sum(ss2);
      if (!__all_sync(FULL, inrange)) st = TF_PRECISION_OVERFLOW;
      double n2 = sqrt(ss2);
      if (!st && n2 < 1e-12) st = TF_DEGENERATE_EMBEDDING;
      __syncwarp();
      if (!st)
        for (int i = lane; i < dim; i += 32) o[i] = static_cast<float>(static_cast<double>(o[i]) / n2);
    }
  }
  if (lane == 0) status[r] = st;
}

__global__ void binary16_kernel(long long n, const float* in, float* out, int* status) {
  long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float v = in[i];
  int st = 0;
  if (!isfinite(v) || fabsf(v) > 65504.0f) st = TF_PRECISION_OVERFLOW;
  out[i] = __half2float(__float2half_rn(v));
  status[i] = st;
}

__global__ void smooth_kernel(int n, int dim, const float* oldv, const float* newv, double alpha, double beta,
                              float* out, int* status) {
  const int r = blockIdx.x * n_warps() + warp_id();
  if (r >= n) return;
  const int lane = lane_id();
  const float* o = oldv + static_cast<long long>(r) * dim;
  const float* q = newv + static_cast<long long>(r) * dim;
  double ss = 0.0;
  bool fin = true;
  for (int i = lane; i < dim; i += 32) {
    double v = alpha * static_cast<double>(o[i]) + beta * static_cast<double>(q[i]);
    fin = fin && isfinite(v);
    ss += v * v;
  }
  ss = warp_sum(ss);
  fin = __all_sync(FULL, fin);
  double nrm = sqrt(ss);
  int st = (!fin || nrm < 1e-12) ? TF_DEGENERATE_EMBEDDING : 0;
  if (!st)
    for (int i = lane; i < dim; i += 32) {
      double v = alpha * static_cast<double>(o[i]) + beta * static_cast<double>(q[i]);
      out[static_cast<long long>(r) * dim + i] = static_cast<float>(v / nrm);
    }
  if (lane == 0) status[r] = st;
}

__global__ void iou_kernel(int n, const double* a, const double* b, double* out) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = iou_tlwh(a[4 * i], a[4 * i + 1], a[4 * i + 2], a[4 * i + 3], b[4 * i], b[4 * i + 1], b[4 * i + 2],
                    b[4 * i + 3]);
}

// ============================================================================
// Host launchers
// ============================================================================

size_t frame_smem_bytes(int total_anchors, int cap_cand) {
  return frame_plan(total_anchors, cap_cand, (cap_cand + 63) / 64).total;
}
size_t assoc_static_smem() {
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, associate_kernel<kAssocThreads, false>) != cudaSuccess) return 8192;
  return fa.sharedSizeBytes;
}

size_t assoc_smem_bytes(int cap_tracks, int cap_det, int cap_entries) {
  return assoc_plan(cap_tracks, cap_det, cap_entries).total;
}

cudaError_t launch_frame_heads(const HeadLaunch& h, const Params& P, cudaStream_t st) {
  FrameArgs a = {};
  for (int i = 0; i < 3; ++i) {
    const tf_head_scale& s = h.heads->scale[i];
    a.sc[i].head = h.head_ptr[i];
    a.sc[i].hs_n = s.head_stride_n;
    a.sc[i].hs_c = s.head_stride_c;
    a.sc[i].delta = h.delta_ptr[i];
    a.sc[i].ds_n = h.delta_stride_n[i];
    a.sc[i].ds_c = h.delta_stride_c[i];
    a.sc[i].emb = h.emb_ptr[i];
    a.sc[i].es_n = s.emb_stride_n;
    a.sc[i].es_c = s.emb_stride_c;
    a.sc[i].es_h = s.emb_stride_h;
    a.sc[i].es_w = s.emb_stride_w;
    a.sc[i].H = s.height;
    a.sc[i].W = s.width;
    a.sc[i].stride = s.stride;
    a.sc[i].pad = 0;
    for (int q = 0; q < 4; ++q) {
      a.sc[i].aw[q] = s.anchors[2 * q];
      a.sc[i].ah[q] = s.anchors[2 * q + 1];
    }
  }
  a.scale_inv = h.heads->scale_inv;
  a.pad_x = h.heads->pad_x;
  a.pad_y = h.heads->pad_y;
  a.frames = h.frames;
  a.cap_cand = h.cap_cand;
  a.cap_det = h.cap_det;
  a.words = (h.cap_cand + 63) / 64;
  a.det = h.det;
  a.ready = h.ready;
  a.epoch = h.epoch;
  a.ticket = h.ticket;
  a.order = h.order;
  a.first_wave = h.first_wave;
  a.streams = h.streams;
  a.B = h.B;
  int total = 0;
  for (int i = 0; i < 3; ++i) total += 4 * h.heads->scale[i].height * h.heads->scale[i].width;
  const size_t smem = frame_smem_bytes(total, h.cap_cand);
  const int sms = sm_count();
  const bool many = h.frames >= 2 * sms;
  int cr = 1;                                      // CTAs per frame (cluster) when frames are few
  if (!many)
    while (cr < 8 && h.frames * cr * 2 <= sms) cr *= 2;
  if (h.ready) cr = 1;                             // overlapped mode: persistent, one CTA per SM slot
  auto go = [&](auto kern, int threads) {
    set_smem(reinterpret_cast<const void*>(kern), smem);
    // overlapped mode: an association CTA (~110 KB of shared memory) must fit
    // next to the decode CTAs on an SM, and an SM only hosts CTAs of kernels
    // whose shared-memory carveout it is configured with, so the decode asks
    // for the maximum carveout too (otherwise the association waits for SMs
    // to drain, i.e. for the end of the decode)
    if (h.ready) {
      static std::mutex mu;
      static std::map<std::pair<const void*, int>, bool> done;
      int dev = 0;
      cudaGetDevice(&dev);
      std::lock_guard<std::mutex> lock(mu);
      auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
      if (!done[key]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
        done[key] = true;
      }
    }
    if (cr == 1) {
      const int grid = h.ready ? std::min(h.frames, h.persist_ctas) : h.frames;
      kern<<<grid, threads, smem, st>>>(a, P);
      return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(h.frames * cr));
    cfg.blockDim = dim3(static_cast<unsigned>(threads));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(cr);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, a, P);
  };
  if (h.heads->dtype == 1) {          // binary16 heads and embedding maps
    if (many) go(frame_heads_kernel<__half, 256>, 256); else go(frame_heads_kernel<__half, 1024>, 1024);
  } else {
    if (many) go(frame_heads_kernel<float, 256>, 256); else go(frame_heads_kernel<float, 1024>, 1024);
  }
  return cudaGetLastError();
}

cudaError_t launch_frame_dets(const double* boxes, const double* obj, const float* emb, const uint8_t* has,
                              int n, int cap_cand, int cap_det, const DetBuf& det, const Params& P,
                              cudaStream_t st) {
  RowsArgs a;
  a.boxes = boxes;
  a.obj = obj;
  a.emb = emb;
  a.has_emb = has;
  a.offsets = nullptr;
  a.n = n;
  a.normalize = 0;
  a.cap_cand = cap_cand;
  a.cap_det = cap_det;
  a.words = (cap_cand + 63) / 64;
  a.det = det;
  const size_t smem = frame_smem_bytes(0, cap_cand);
  set_smem(reinterpret_cast<const void*>(frame_dets_kernel), smem);
  frame_dets_kernel<<<1, 512, smem, st>>>(a, P);
  return cudaGetLastError();
}

cudaError_t launch_frame_rows(const double* boxes, const double* obj, const float* emb, const int* offsets,
                              int frames, int normalize, int cap_cand, int cap_det, const DetBuf& det,
                              const Params& P, cudaStream_t st) {
  RowsArgs a;
  a.boxes = boxes;
  a.obj = obj;
  a.emb = emb;
  a.has_emb = nullptr;
  a.offsets = offsets;
  a.n = 0;
  a.normalize = normalize;
  a.cap_cand = cap_cand;
  a.cap_det = cap_det;
  a.words = (cap_cand + 63) / 64;
  a.det = det;
  const size_t smem = frame_smem_bytes(0, cap_cand);
  set_smem(reinterpret_cast<const void*>(frame_dets_kernel), smem);
  frame_dets_kernel<<<frames, 512, smem, st>>>(a, P);
  return cudaGetLastError();
}

template <bool kExt>
static cudaError_t launch_associate_t(const AssocArgs& a, int n_streams, const Params& P, cudaStream_t st) {
#ifdef TF_CANARY
  const size_t smem = assoc_smem_bytes(a.cap_tracks, a.cap_det, a.cap_entries) + 256;
#else
  const size_t smem = assoc_smem_bytes(a.cap_tracks, a.cap_det, a.cap_entries);
#endif
  if (a.threads == kAssocThreadsSmall) {
    set_smem(reinterpret_cast<const void*>(associate_kernel<kAssocThreadsSmall, kExt>), smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(n_streams));
    cfg.blockDim = dim3(kAssocThreadsSmall);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, associate_kernel<kAssocThreadsSmall, kExt>, a, P);
  }
  set_smem(reinterpret_cast<const void*>(associate_kernel<kAssocThreads, kExt>), smem);
  if (a.cluster <= 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(n_streams));
    cfg.blockDim = dim3(kAssocThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // see griddepcontrol in the kernel
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, associate_kernel<kAssocThreads, kExt>, a, P);
  }
  if (kExt && a.cluster > 8) {          // (the reference-path instantiation is set up by assoc_cluster_size)
    static bool nonportable = false;
    if (!nonportable)
      cudaFuncSetAttribute(associate_kernel<kAssocThreads, kExt>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    nonportable = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(n_streams * a.cluster));
  cfg.blockDim = dim3(kAssocThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(a.cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, associate_kernel<kAssocThreads, kExt>, a, P);
}

cudaError_t launch_associate(const AssocArgs& a, int n_streams, const Params& P, cudaStream_t st) {
  return (P.fuse || P.iou_stage) ? launch_associate_t<true>(a, n_streams, P, st)
                                 : launch_associate_t<false>(a, n_streams, P, st);
}

int assoc_cluster_size(int n_streams, int cap_tracks, int cap_det, int cap_entries) {
  // One stream per cluster; followers only help in the parallel phases, so
  // spread few streams over up to 16 SMs each, never beyond the SM count.
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // 16 (non-portable) when the streams leave room: the cost phase scales with
  // the number of follower warps (B200: 31.9k -> 33.5k frames/s at cfg1)
  const char* env = getenv("TF_CLUSTER");
  int c = 16;
  if (env) c = atoi(env);
  if (c > 16) c = 16;
  while (c > 1 && n_streams * c > sms) c >>= 1;
  if (c > 1) {
    const size_t smem = assoc_smem_bytes(cap_tracks, cap_det, cap_entries);
    set_smem(reinterpret_cast<const void*>(associate_kernel<kAssocThreads, false>), smem);   // (only ever raised: see set_smem)
    if (c > 8) cudaFuncSetAttribute(associate_kernel<kAssocThreads, false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(c));
    cfg.blockDim = dim3(kAssocThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = static_cast<unsigned>(c);
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // every stream's cluster must be resident at once (clusters live inside a
    // GPC; a second wave would double the update time): shrink until they fit
    int clusters = 0;
    while (c > 1 && (cudaOccupancyMaxActiveClusters(&clusters, associate_kernel<kAssocThreads, false>, &cfg) != cudaSuccess ||
                     clusters < n_streams)) {
      c >>= 1;
      cfg.gridDim = dim3(static_cast<unsigned>(c));
      attr[0].val.clusterDim.x = static_cast<unsigned>(c);
    }
    cudaGetLastError();
  }
  return c < 1 ? 1 : c;
}

cudaError_t launch_nms_sets(int n_sets, const int* offsets, const double* boxes, const double* scores,
                            const double* thr, uint8_t* keep, int* status, int cap, cudaStream_t st) {
  const int words = (cap + 63) / 64;
  const size_t smem = frame_smem_bytes(0, cap);
  cudaFuncSetAttribute(nms_sets_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  nms_sets_kernel<<<n_sets, 256, smem, st>>>(offsets, boxes, scores, thr, keep, status, cap, words);
  return cudaGetLastError();
}

cudaError_t launch_lap_dense(int n, const int* shapes, const long long* cost_off, const double* costs,
                             const long long* row_off, int* col_for_row, int* status, int cap_n,
                             int16_t* pool_col, double* pool_val, int* pool_rowptr, long long pool_stride,
                             cudaStream_t st) {
  const size_t smem = 32 * static_cast<size_t>(cap_n) + 12 * static_cast<size_t>(cap_n) + 64;
  cudaFuncSetAttribute(lap_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  lap_dense_kernel<<<n, 32, smem, st>>>(shapes, cost_off, costs, row_off, col_for_row, status, cap_n, pool_col,
                                        pool_val, pool_rowptr, pool_stride);
  return cudaGetLastError();
}

cudaError_t launch_kalman(int op, int n, const Params& P, const double* mi, const double* ci, const double* z,
                          double* mo, double* co, int* status, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const size_t smem = ((op == 1 || op == 3) ? 1 : 2) * sizeof(double) * kKfBlock * kKfPad;
  cudaFuncSetAttribute(kalman_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  kalman_kernel<<<(n + kKfBlock - 1) / kKfBlock, kKfBlock, smem, st>>>(op, n, P, mi, ci, z, mo, co, status);
  return cudaGetLastError();
}

cudaError_t launch_gating(int nt, const double* means, const double* covs, int nm, const double* z, int metric,
                          const Params& P, double* out, int* status, cudaStream_t st) {
  if (nt == 0) return cudaSuccess;
  gating_kernel<<<nt, 128, 0, st>>>(nt, means, covs, nm, z, metric, P, out, status);
  return cudaGetLastError();
}

cudaError_t launch_cosine_cost(int nt, int nd, int dim, const float* te, const float* de, double* out,
                               cudaStream_t st) {
  const int pairs = nt * nd;
  if (pairs == 0) return cudaSuccess;
  cosine_cost_kernel<<<(pairs + 7) / 8, 256, 0, st>>>(nt, nd, dim, te, de, out);
  return cudaGetLastError();
}

cudaError_t launch_normalize_rows(int n, int dim, const double* in64, const float* in32, long long stride,
                                  int quantize, float* out, int* status, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  normalize_rows_kernel<<<(n + 7) / 8, 256, 0, st>>>(n, dim, in64, in32, stride, quantize, out, status);
  return cudaGetLastError();
}

cudaError_t launch_binary16(long long n, const float* in, float* out, int* status, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  binary16_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(n, in, out, status);
  return cudaGetLastError();
}

cudaError_t launch_smooth(int n, int dim, const float* o, const float* q, double alpha, double beta, float* out,
                          int* status, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  smooth_kernel<<<(n + 7) / 8, 256, 0, st>>>(n, dim, o, q, alpha, beta, out, status);
  return cudaGetLastError();
}

cudaError_t launch_iou(int n, const double* a, const double* b, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  iou_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, a, b, out);
  return cudaGetLastError();
}

}  // namespace tfd
