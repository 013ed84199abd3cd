// sm_100a kernels of the MOT evaluation of tracker outputs (SURVEY.md 8(f)
// row 3): tf/moteval.py restated on the device.
//
//  mot_accumulate_kernel  one CTA per sequence, frames in order: the carry-over
//                         of last frame's (gt -> hyp) pairs, the IoU cost of
//                         the remaining pairs and the scipy-order LAP of
//                         hungarian_solve (warp_lap_fast) -- match_frame +
//                         accumulate, tf/moteval.py:36-110.
//  mot_coverage_kernel    one CTA per frame: joint coverage counts of every
//                         (gt trajectory, hyp trajectory) pair for the identity
//                         metrics, tf/moteval.py:196-232,337-345.
//
// Ids are dense indices (the host maps them); boxes are tlwh fp64; IoU is the
// reference's expression (iou_tlwh, tf/core.py:71-80).

#include "tf_kernels.cuh"

namespace tfd {

namespace {

constexpr int kMotThreads = 128;

struct MotPlan {
  size_t off_takeg, off_takeh, off_freeg, off_freeh, off_rowptr, off_col, off_val, off_u, off_v, off_dist, off_crow,
      off_path, off_r4c, off_c4r, off_rem, off_vr, off_vc, total;
};

__host__ __device__ inline size_t a16(size_t v) { return (v + 15) & ~size_t(15); }

__host__ __device__ inline MotPlan mot_plan(int cap_g, int cap_h, int cap_e) {
  MotPlan p;
  const int n = cap_g > cap_h ? cap_g : cap_h;
  size_t o = 0;
#define TF_TAKE(field, bytes) p.field = o; o = a16(o + (bytes));
  TF_TAKE(off_takeg, cap_g)
  TF_TAKE(off_takeh, cap_h)
  TF_TAKE(off_freeg, 2 * cap_g)
  TF_TAKE(off_freeh, 2 * cap_h)
  TF_TAKE(off_rowptr, 4 * (cap_g + 1))
  TF_TAKE(off_col, 2 * cap_e)
  TF_TAKE(off_val, 8 * cap_e)
  TF_TAKE(off_u, 8 * n)
  TF_TAKE(off_v, 8 * n)
  TF_TAKE(off_dist, 8 * n)
  TF_TAKE(off_crow, 8 * n)
  TF_TAKE(off_path, 2 * n)
  TF_TAKE(off_r4c, 2 * n)
  TF_TAKE(off_c4r, 2 * n)
  TF_TAKE(off_rem, 2 * n)
  TF_TAKE(off_vr, 2 * (2 * n + 1))
  TF_TAKE(off_vc, 2 * (2 * n + 1))
#undef TF_TAKE
  p.total = o;
  return p;
}

struct MotSeq {
  const int* gt_ptr;      // [F + 1] rows of frame f
  const int* gt_id;       // dense gt id per row
  const double* gt_box;   // [rows][4] tlwh
  const int* hyp_ptr;
  const int* hyp_id;
  const double* hyp_box;
  int frames, cap_g, cap_h, cap_e;
  double iou_min;
  int* prev;              // [n_gt_ids] last matched dense hyp id, -1 (workspace)
  int* hpos;              // [n_hyp_ids] row of the hyp id in the current frame, -1 (workspace)
  int n_gt_ids, n_hyp_ids;
  // outputs
  int* match_count;       // [F]
  int* match_gt;          // [gt rows] match i of frame f at gt_ptr[f] + i: gt row
  int* match_hyp;         //   ... hyp row
  double* match_iou;      //   ... overlap (1 - cost for assignment matches, as the reference)
  uint8_t* gt_matched;    // [gt rows]
  uint8_t* hyp_matched;   // [hyp rows]
  int* status;
};

__device__ inline double box_iou(const double* a, const double* b) {
  return iou_tlwh(a[0], a[1], a[2], a[3], b[0], b[1], b[2], b[3]);
}

__global__ void __launch_bounds__(kMotThreads) mot_accumulate_kernel(MotSeq q) {
  extern __shared__ __align__(16) unsigned char smem[];
  const MotPlan pl = mot_plan(q.cap_g, q.cap_h, q.cap_e);
  uint8_t* take_g = smem + pl.off_takeg;
  uint8_t* take_h = smem + pl.off_takeh;
  int16_t* free_g = reinterpret_cast<int16_t*>(smem + pl.off_freeg);
  int16_t* free_h = reinterpret_cast<int16_t*>(smem + pl.off_freeh);
  int* rowptr = reinterpret_cast<int*>(smem + pl.off_rowptr);
  int16_t* ecol = reinterpret_cast<int16_t*>(smem + pl.off_col);
  double* eval = reinterpret_cast<double*>(smem + pl.off_val);
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
  __shared__ int s_n[4];   // n matched (carry-over), free gt, free hyp, entries
  __shared__ double s_amp;
  __shared__ int s_err;
  const int tid = threadIdx.x, lane = lane_id(), wid = warp_id();
  for (int i = tid; i < q.n_gt_ids; i += blockDim.x) q.prev[i] = -1;
  for (int i = tid; i < q.n_hyp_ids; i += blockDim.x) q.hpos[i] = -1;
  if (tid == 0) s_err = 0;
  __syncthreads();
  for (int f = 0; f < q.frames; ++f) {
    const int g0 = q.gt_ptr[f], G = q.gt_ptr[f + 1] - g0;
    const int h0 = q.hyp_ptr[f], H = q.hyp_ptr[f + 1] - h0;
    if (G > q.cap_g || H > q.cap_h) {
      if (tid == 0) s_err = TF_CAPACITY;
      break;
    }
    for (int j = tid; j < H; j += blockDim.x) {
      q.hpos[q.hyp_id[h0 + j]] = j;
      take_h[j] = 0;
    }
    for (int i = tid; i < G; i += blockDim.x) take_g[i] = 0;
    __syncthreads();
    // carry-over of last frame's pairs, in gt order (tf/moteval.py:58-67)
    if (tid == 0) {
      int nm = 0;
      for (int i = 0; i < G; ++i) {
        const int h = q.prev[q.gt_id[g0 + i]];
        if (h < 0) continue;
        const int j = q.hpos[h];
        if (j < 0 || take_h[j]) continue;
        const double ov = box_iou(q.gt_box + 4LL * (g0 + i), q.hyp_box + 4LL * (h0 + j));
        if (ov >= q.iou_min) {
          q.match_gt[g0 + nm] = g0 + i;
          q.match_hyp[g0 + nm] = h0 + j;
          q.match_iou[g0 + nm] = ov;
          ++nm;
          take_g[i] = 1;
          take_h[j] = 1;
        }
      }
      int ng = 0, nh = 0;
      for (int i = 0; i < G; ++i)
        if (!take_g[i]) free_g[ng++] = static_cast<int16_t>(i);
      for (int j = 0; j < H; ++j)
        if (!take_h[j]) free_h[nh++] = static_cast<int16_t>(j);
      s_n[0] = nm;
      s_n[1] = ng;
      s_n[2] = nh;
      s_amp = 0.0;
    }
    __syncthreads();
    const int nm = s_n[0], ng = s_n[1], nh = s_n[2];
    // IoU cost of the free pairs, forbidden below iou_min (tf/moteval.py:69-77):
    // one thread per free gt row counts, a warp scan places, the row fills
    for (int r = tid; r < ng; r += blockDim.x) {
      const double* gb = q.gt_box + 4LL * (g0 + free_g[r]);
      int c = 0;
      for (int k = 0; k < nh; ++k) c += box_iou(gb, q.hyp_box + 4LL * (h0 + free_h[k])) >= q.iou_min;
      rowptr[r + 1] = c;
    }
    __syncthreads();
    if (wid == 0) {
      int carry = 0;
      if (lane == 0) rowptr[0] = 0;
      for (int r0 = 0; r0 < ng; r0 += 32) {
        const int r = r0 + lane;
        const int v = r < ng ? rowptr[r + 1] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(FULL, incl, o);
          if (lane >= o) incl += t;
        }
        __syncwarp();
        if (r < ng) rowptr[r + 1] = carry + incl;
        carry += __shfl_sync(FULL, incl, 31);
      }
      if (lane == 0) s_n[3] = carry;
    }
    __syncthreads();
    if (s_n[3] > q.cap_e) {
      if (tid == 0) s_err = TF_CAPACITY;
      break;
    }
    for (int r = tid; r < ng; r += blockDim.x) {
      const double* gb = q.gt_box + 4LL * (g0 + free_g[r]);
      int e = rowptr[r];
      double amp = 0.0;
      for (int k = 0; k < nh; ++k) {
        const double ov = box_iou(gb, q.hyp_box + 4LL * (h0 + free_h[k]));
        if (ov >= q.iou_min) {
          ecol[e] = static_cast<int16_t>(k);
          eval[e] = 1.0 - ov;
          amp = fmax(amp, fabs(1.0 - ov));
          ++e;
        }
      }
      if (amp > 0.0) atomicMax(reinterpret_cast<unsigned long long*>(&s_amp),
                               static_cast<unsigned long long>(__double_as_longlong(amp)));
    }
    __syncthreads();
    // hungarian_solve (tf/assoc.py:60-87): sentinel-padded square matrix, scipy order
    if (wid == 0 && ng > 0 && nh > 0) {
      const int n = ng > nh ? ng : nh;
      const double amp = s_n[3] > 0 ? s_amp : 1.0;
      const double sentinel = 2.0 * static_cast<double>(n) * fmax(amp, 1.0) + 1.0;
      warp_lap_fast(n, ng, CsrRows{rowptr, ecol, eval}, sentinel, L);
      __syncwarp();
      if (lane == 0) {
        int k = nm;
        for (int r = 0; r < ng; ++r) {
          const int c = L.col4row[r];
          if (c >= nh) continue;
          for (int e = rowptr[r]; e < rowptr[r + 1]; ++e)
            if (ecol[e] == c) {
              const int i = free_g[r], j = free_h[c];
              q.match_gt[g0 + k] = g0 + i;
              q.match_hyp[g0 + k] = h0 + j;
              q.match_iou[g0 + k] = 1.0 - eval[e];
              take_g[i] = 1;
              take_h[j] = 1;
              ++k;
              break;
            }
        }
        s_n[0] = k;
      }
    }
    __syncthreads();
    const int nmatch = s_n[0];
    for (int m = tid; m < nmatch; m += blockDim.x)
      q.prev[q.gt_id[q.match_gt[g0 + m]]] = q.hyp_id[q.match_hyp[g0 + m]];
    for (int i = tid; i < G; i += blockDim.x) q.gt_matched[g0 + i] = take_g[i];
    for (int j = tid; j < H; j += blockDim.x) {
      q.hyp_matched[h0 + j] = take_h[j];
      q.hpos[q.hyp_id[h0 + j]] = -1;
    }
    if (tid == 0) q.match_count[f] = nmatch;
    __syncthreads();
  }
  if (tid == 0) *q.status = s_err;
}

// Joint coverage of trajectory pairs: one CTA per frame, every (gt, hyp) pair
// of the frame with IoU >= iou_min adds one to coverage[gt id][hyp id].
__global__ void __launch_bounds__(kMotThreads) mot_coverage_kernel(const int* gt_ptr, const int* gt_id,
                                                                   const double* gt_box, const int* hyp_ptr,
                                                                   const int* hyp_id, const double* hyp_box,
                                                                   double iou_min, int n_hyp_ids, int* coverage) {
  const int f = blockIdx.x;
  const int g0 = gt_ptr[f], G = gt_ptr[f + 1] - g0;
  const int h0 = hyp_ptr[f], H = hyp_ptr[f + 1] - h0;
  for (int x = threadIdx.x; x < G * H; x += blockDim.x) {
    const int i = x / H, j = x - i * H;
    if (box_iou(gt_box + 4LL * (g0 + i), hyp_box + 4LL * (h0 + j)) >= iou_min)
      atomicAdd(&coverage[static_cast<long long>(gt_id[g0 + i]) * n_hyp_ids + hyp_id[h0 + j]], 1);
  }
}

}  // namespace

size_t mot_accumulate_smem(int cap_g, int cap_h, int cap_e) { return mot_plan(cap_g, cap_h, cap_e).total; }

cudaError_t launch_mot_accumulate(int frames, const int* gt_ptr, const int* gt_id, const double* gt_box,
                                  const int* hyp_ptr, const int* hyp_id, const double* hyp_box, int n_gt_ids,
                                  int n_hyp_ids, double iou_min, int cap_g, int cap_h, int cap_e, int* prev, int* hpos,
                                  int* match_count, int* match_gt, int* match_hyp, double* match_iou,
                                  uint8_t* gt_matched, uint8_t* hyp_matched, int* status, cudaStream_t st) {
  MotSeq q;
  q.gt_ptr = gt_ptr; q.gt_id = gt_id; q.gt_box = gt_box;
  q.hyp_ptr = hyp_ptr; q.hyp_id = hyp_id; q.hyp_box = hyp_box;
  q.frames = frames; q.cap_g = cap_g; q.cap_h = cap_h; q.cap_e = cap_e;
  q.iou_min = iou_min;
  q.prev = prev; q.hpos = hpos;
  q.n_gt_ids = n_gt_ids; q.n_hyp_ids = n_hyp_ids;
  q.match_count = match_count; q.match_gt = match_gt; q.match_hyp = match_hyp; q.match_iou = match_iou;
  q.gt_matched = gt_matched; q.hyp_matched = hyp_matched; q.status = status;
  const size_t smem = mot_plan(cap_g, cap_h, cap_e).total;
  cudaFuncSetAttribute(mot_accumulate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  mot_accumulate_kernel<<<1, kMotThreads, smem, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_mot_coverage(int frames, const int* gt_ptr, const int* gt_id, const double* gt_box,
                                const int* hyp_ptr, const int* hyp_id, const double* hyp_box, double iou_min,
                                int n_hyp_ids, int* coverage, cudaStream_t st) {
  if (frames == 0) return cudaSuccess;
  mot_coverage_kernel<<<frames, kMotThreads, 0, st>>>(gt_ptr, gt_id, gt_box, hyp_ptr, hyp_id, hyp_box, iou_min,
                                                      n_hyp_ids, coverage);
  return cudaGetLastError();
}

}  // namespace tfd

// ---- C ABI ------------------------------------------------------------------

extern "C" {

int tf_mot_accumulate(int32_t n_frames, const int32_t* gt_ptr, const int32_t* gt_id, const double* gt_box,
                      const int32_t* hyp_ptr, const int32_t* hyp_id, const double* hyp_box, int32_t n_gt_ids,
                      int32_t n_hyp_ids, int32_t max_gt_per_frame, int32_t max_hyp_per_frame,
                      int32_t max_pairs_per_frame, double iou_min, int32_t* match_count, int32_t* match_gt,
                      int32_t* match_hyp, double* match_iou, uint8_t* gt_matched, uint8_t* hyp_matched,
                      int32_t* status, void* cuda_stream) {
  if (n_frames < 0 || n_gt_ids < 0 || n_hyp_ids < 0) return TF_ARGUMENT;
  if (n_frames == 0) return TF_OK;
  if (!gt_ptr || !hyp_ptr || !match_count || !status) return TF_ARGUMENT;
  const int cap_g = max_gt_per_frame > 0 ? max_gt_per_frame : 1;
  const int cap_h = max_hyp_per_frame > 0 ? max_hyp_per_frame : 1;
  const int cap_e = max_pairs_per_frame > 0 ? max_pairs_per_frame : 1;
  if (cap_g > 32767 || cap_h > 32767 || cap_e > 32767) return TF_CAPACITY;
  int optin = 0, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (tfd::mot_accumulate_smem(cap_g, cap_h, cap_e) + 1024 > static_cast<size_t>(optin)) return TF_CAPACITY;
  cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
  int *prev = nullptr, *hpos = nullptr;
  if (cudaMallocAsync(&prev, sizeof(int) * (n_gt_ids + 1), st) != cudaSuccess ||
      cudaMallocAsync(&hpos, sizeof(int) * (n_hyp_ids + 1), st) != cudaSuccess)
    return TF_CUDA;
  cudaError_t e = tfd::launch_mot_accumulate(n_frames, gt_ptr, gt_id, gt_box, hyp_ptr, hyp_id, hyp_box, n_gt_ids,
                                             n_hyp_ids, iou_min, cap_g, cap_h, cap_e, prev, hpos, match_count,
                                             match_gt, match_hyp, match_iou, gt_matched, hyp_matched, status, st);
  cudaFreeAsync(prev, st);
  cudaFreeAsync(hpos, st);
  return e == cudaSuccess ? TF_OK : TF_CUDA;
}

int tf_mot_coverage(int32_t n_frames, const int32_t* gt_ptr, const int32_t* gt_id, const double* gt_box,
                    const int32_t* hyp_ptr, const int32_t* hyp_id, const double* hyp_box, int32_t n_hyp_ids,
                    double iou_min, int32_t* coverage, void* cuda_stream) {
  if (n_frames < 0 || n_hyp_ids < 0) return TF_ARGUMENT;
  if (n_frames == 0) return TF_OK;
  if (!gt_ptr || !hyp_ptr || !coverage) return TF_ARGUMENT;
  cudaError_t e = tfd::launch_mot_coverage(n_frames, gt_ptr, gt_id, gt_box, hyp_ptr, hyp_id, hyp_box, iou_min,
                                           n_hyp_ids, coverage, static_cast<cudaStream_t>(cuda_stream));
  return e == cudaSuccess ? TF_OK : TF_CUDA;
}

}  // extern "C"
