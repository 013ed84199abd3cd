// Device building blocks of the decode -> NMS -> association path (sm_100a).
//
// Precision policy: every value that feeds a decision
// (confidence test, IoU > thr, gate > thr, cost > max_cost, LAP costs) is
// computed in fp64 with the reference's operation order, so decisions match
// the CPU reference bit for bit. The translation unit is compiled with
// --fmad=false so no a*b+c is silently contracted into an FMA.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <math.h>

#include "../../include/trackforge_b200.h"

namespace tfd {

constexpr unsigned FULL = 0xffffffffu;

// Host-prepared constants (tf_config + derived values computed once on the host).
struct Params {
  double conf_threshold;   // filter_confidence  (tf/postproc.py:61-65)
  double conf_logit;       // logit(conf_threshold): exact logit-space pre-filter of the decode
  double nms_iou;          // tf/postproc.py:68-89
  double max_cost;         // tf/assoc.py:90-107
  double gate_threshold;   // tf/assoc.py:49-57
  double alpha, beta;      // smoothing alpha and (1.0 - alpha) as Python computes it
  double wp, wv;           // MotionNoise weights (tf/motion.py:37-38)
  double std_aspect, std_aspect_velocity, std_aspect_measurement;
  int gate_metric;         // 0 mahalanobis, 1 euclidean, other -> ConfigError when used
  int max_lost, min_hits, dim, quantize;
  // JDE extensions (off = the reference): lambda-fused cost and a second
  // association stage on 1 - IoU
  double lambda, lambda_w;  // cost = lambda * cosine + lambda_w * gate distance when fuse
  double iou_threshold;
  int fuse, iou_stage;
};

// ---------------------------------------------------------------- misc
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int n_warps() { return blockDim.x >> 5; }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

// Order-preserving map of a double onto uint64 (for min-reductions).
__device__ __forceinline__ unsigned long long dkey(double d) {
  long long b = __double_as_longlong(d + 0.0);  // canonicalise -0.0
  return (b < 0) ? ~static_cast<unsigned long long>(b)
                 : (static_cast<unsigned long long>(b) | 0x8000000000000000ull);
}

// Record the first error (lowest packed key) in a status word. Key packs
// (position << 8 | code) so the earliest failing row / frame wins.
__device__ __forceinline__ void flag_error(int* status, int position, int code) {
  atomicMin(status, (position << 8) | code);
}
constexpr int STATUS_CLEAR = 0x7fffffff;

// a / b in round-to-nearest from y = RN(1/b) (__drcp_rn): q0 = RN(a*y), the
// remainder a - b*q0 is exact by FMA, and RN(q0 + rem*y) is the correctly
// rounded quotient (Markstein's theorem; no overflow / underflow for the
// unit-vector magnitudes it is used on). One reciprocal serves many
// divisions by the same norm; tests/test_gpu_units.py checks it against
// true division.
__device__ __forceinline__ double div_by(double a, double b, double y) {
  const double q0 = a * y;
  const double r = fma(-b, q0, a);
  return fma(r, y, q0);
}

// ---------------------------------------------------------------- geometry
// iou, tf/core.py:71-80 (right = x + w, bottom = y + h, area = w * h; clamp to 1).
__device__ __forceinline__ double iou_tlwh(double ax, double ay, double aw, double ah,
                                           double bx, double by, double bw, double bh) {
  double iw = fmin(ax + aw, bx + bw) - fmax(ax, bx);
  double ih = fmin(ay + ah, by + bh) - fmax(ay, by);
  if (iw <= 0.0 || ih <= 0.0) return 0.0;
  double inter = iw * ih;
  double uni = (aw * ah + bw * bh) - inter;
  return fmin(inter / uni, 1.0);
}

// box_to_measurement, tf/core.py:83-88.
__device__ __forceinline__ void box_to_meas(const double* b, double* m) {
  m[0] = b[0] + b[2] / 2.0;
  m[1] = b[1] + b[3] / 2.0;
  m[2] = b[2] / b[3];
  m[3] = b[3];
}

// measurement_to_box + BoundingBox validation, tf/core.py:91-97, 37-43.
// Returns false (InvalidBoxError) on non-positive or non-finite size.
__device__ __forceinline__ bool meas_to_box(const double* m, double* b) {
  double cx = m[0], cy = m[1], a = m[2], h = m[3];
  double w = a * h;
  if (!(h > 0.0) || !(w > 0.0)) return false;
  b[0] = cx - w / 2.0;
  b[1] = cy - h / 2.0;
  b[2] = w;
  b[3] = h;
  return isfinite(b[0]) && isfinite(b[1]) && isfinite(b[2]) && isfinite(b[3]);
}

// ---------------------------------------------------------------- Kalman (compact)
// The reference filter (tf/motion.py) keeps an 8x8 covariance, but starting
// from initiate()'s diagonal every predict/update only ever couples state i
// with i+4: the filter is four independent (position, velocity) pairs and the
// innovation covariance S is exactly diagonal. We store per axis i
// (pp, pv, vv) = (P[i][i], P[i][i+4], P[i+4][i+4]) and reproduce each
// reference operation with its rounding order:
//   predict: F P F^T + diag(q) then symmetrise      (tf/motion.py:83-101)
//   project: S_i = P_ii + r_i^2                     (tf/motion.py:103-110)
//   update : Cholesky of diagonal S, gain = (P H^T) * (1/l) * (1/l) -- LAPACK
//            trsm multiplies by the reciprocal diagonal -- then
//            P - (K S) K^T and symmetrise          (tf/motion.py:112-126)
//   gate   : sum_i ((z_i - m_i) * (1/l_i))^2 summed in order i = 0..3
//                                                   (tf/motion.py:128-142)
struct KF {
  // process-noise std of axis i (position block), tf/motion.py:87-98
  __device__ static __forceinline__ double qpos(const Params& p, int i, double h) {
    return i == 2 ? p.std_aspect : p.wp * h;
  }
  __device__ static __forceinline__ double qvel(const Params& p, int i, double h) {
    return i == 2 ? p.std_aspect_velocity : p.wv * h;
  }
  __device__ static __forceinline__ double rstd(const Params& p, int i, double h) {
    return i == 2 ? p.std_aspect_measurement : p.wp * h;
  }

  // initiate, tf/motion.py:61-81. mean[8], cov[12] (per axis pp, pv, vv).
  __device__ static __forceinline__ void initiate(const Params& p, const double* z, double* mean,
                                                  double* cov) {
    double h = z[3];
    double wp2 = 2.0 * p.wp, wv10 = 10.0 * p.wv;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      mean[i] = z[i];
      mean[i + 4] = 0.0;
      double sp = (i == 2) ? p.std_aspect : wp2 * h;
      double sv = (i == 2) ? p.std_aspect_velocity : wv10 * h;
      cov[3 * i + 0] = sp * sp;
      cov[3 * i + 1] = 0.0;
      cov[3 * i + 2] = sv * sv;
    }
  }

  __device__ static __forceinline__ void predict(const Params& p, double* mean, double* cov) {
    double h = mean[3];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double qp = qpos(p, i, h), qv = qvel(p, i, h);
      double pp = cov[3 * i], pv = cov[3 * i + 1], vv = cov[3 * i + 2];
      double fpp = pp + pv;          // (F P)[i][i]
      double fpv = pv + vv;          // (F P)[i][i+4] == (F P F^T)[i][i+4]
      cov[3 * i + 0] = (fpp + fpv) + qp * qp;
      cov[3 * i + 1] = fpv;
      cov[3 * i + 2] = vv + qv * qv;
      mean[i] = mean[i] + mean[i + 4];
    }
  }

  // Innovation variances S_i and reciprocal Cholesky factors 1/sqrt(S_i).
  // Returns false when S is not positive definite (NumericError).
  __device__ static __forceinline__ bool project(const Params& p, const double* mean,
                                                 const double* cov, double* s, double* il) {
    double h = mean[3];
    bool ok = true;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double r = rstd(p, i, h);
      s[i] = cov[3 * i] + r * r;
      ok = ok && (s[i] > 0.0);
      il[i] = 1.0 / sqrt(s[i]);
    }
    return ok;
  }

  __device__ static __forceinline__ double mahalanobis(const double* mean, const double* il,
                                                       const double* z) {
    double x0 = (z[0] - mean[0]) * il[0];
    double x1 = (z[1] - mean[1]) * il[1];
    double x2 = (z[2] - mean[2]) * il[2];
    double x3 = (z[3] - mean[3]) * il[3];
    return ((x0 * x0 + x1 * x1) + x2 * x2) + x3 * x3;
  }

  __device__ static __forceinline__ bool update(const Params& p, double* mean, double* cov,
                                                const double* z) {
    double s[4], il[4];
    if (!project(p, mean, cov, s, il)) return false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      double pp = cov[3 * j], pv = cov[3 * j + 1], vv = cov[3 * j + 2];
      double kp = (pp * il[j]) * il[j];
      double kv = (pv * il[j]) * il[j];
      double y = z[j] - mean[j];
      mean[j] = mean[j] + kp * y;
      mean[j + 4] = mean[j + 4] + kv * y;
      double ksp = kp * s[j], ksv = kv * s[j];
      double a = pv - ksp * kv;      // [j][j+4]
      double b = pv - ksv * kp;      // [j+4][j]
      cov[3 * j + 0] = pp - ksp * kp;
      cov[3 * j + 2] = vv - ksv * kv;
      cov[3 * j + 1] = (a + b) / 2.0;
    }
    return true;
  }
};

// ---------------------------------------------------------------- block NMS
// nms, tf/postproc.py:68-89, over C <= cap candidates held in shared memory.
// Greedy order is (-score, index); a candidate is suppressed when its IoU with
// an earlier kept one is strictly above thr. Bitmask formulation: mask[u] has
// bit v set when sorted[v] (v > u) overlaps sorted[u]; one warp then walks the
// sorted order OR-ing masks of kept rows.
//  box   [C*4] tlwh, score [C], alive [C] (filter_confidence result)
//  keep  [C] out: 1 survivor / 0 not
//  sorted [C] int16 scratch; mask [C * words] u64 scratch (words = ceil(cap/64))
// Returns the number of alive candidates. All threads must call.
__device__ inline int block_nms(int C, const double* box, const double* score, const uint8_t* alive,
                         double thr, int16_t* sorted, unsigned long long* mask, int words,
                         uint8_t* keep, int* sh_scratch) {
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) sh_scratch[0] = 0;
  __syncthreads();
  int my_alive = 0;
  for (int i = tid; i < C; i += nt) {
    keep[i] = 0;
    if (!alive[i]) continue;
    ++my_alive;
    double si = score[i];
    int r = 0;
    for (int j = 0; j < C; ++j) {
      if (!alive[j]) continue;
      double sj = score[j];
      r += (sj > si) || (sj == si && j < i);
    }
    sorted[r] = static_cast<int16_t>(i);
  }
  if (my_alive) atomicAdd(sh_scratch, my_alive);
  __syncthreads();
  const int na = sh_scratch[0];
  const int nwords = (na + 63) >> 6;
  const int lane = lane_id(), wid = warp_id(), nw = n_warps();
  for (int u = wid; u < na; u += nw) {
    const int iu = sorted[u];
    const double ax = box[4 * iu], ay = box[4 * iu + 1], aw = box[4 * iu + 2], ah = box[4 * iu + 3];
    for (int w = 0; w < nwords; ++w) {
      unsigned lohi[2];
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        int v = w * 64 + half * 32 + lane;
        bool hit = false;
        if (v > u && v < na) {
          int iv = sorted[v];
          hit = iou_tlwh(ax, ay, aw, ah, box[4 * iv], box[4 * iv + 1], box[4 * iv + 2],
                         box[4 * iv + 3]) > thr;
        }
        lohi[half] = __ballot_sync(FULL, hit);
      }
      if (lane == 0)
        mask[u * words + w] = static_cast<unsigned long long>(lohi[0]) |
                              (static_cast<unsigned long long>(lohi[1]) << 32);
    }
  }
  __syncthreads();
  if (wid == 0 && na <= 64) {
    // Greedy order resolved in parallel (up to 64 boxes, two per lane): box u
    // is kept iff no KEPT box before it suppresses it. Undecided boxes whose
    // suppressors are all decided settle each pass, so the passes follow the
    // longest suppression chain (1-3 in practice) instead of na serial steps.
    unsigned long long in[2] = {0ull, 0ull};         // suppressors of boxes lane, lane + 32
    for (int v = 0; v < na; ++v) {
      const unsigned long long row = mask[v * words];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = lane + 32 * h;
        if (v < u && ((row >> u) & 1ull)) in[h] |= 1ull << v;
      }
    }
    const unsigned long long all = na == 64 ? ~0ull : (1ull << na) - 1ull;
    unsigned long long kept = 0ull, supp = 0ull;
    while ((kept | supp) != all) {
      bool k[2], q[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int u = lane + 32 * h;
        const bool open = u < na && !(((kept | supp) >> u) & 1ull);
        q[h] = open && (in[h] & kept) != 0ull;
        k[h] = open && !q[h] && (in[h] & ~supp) == 0ull;
      }
      kept |= static_cast<unsigned long long>(__ballot_sync(FULL, k[0])) |
              (static_cast<unsigned long long>(__ballot_sync(FULL, k[1])) << 32);
      supp |= static_cast<unsigned long long>(__ballot_sync(FULL, q[0])) |
              (static_cast<unsigned long long>(__ballot_sync(FULL, q[1])) << 32);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int u = lane + 32 * h;
      if (u < na && ((kept >> u) & 1ull)) keep[sorted[u]] = 1;
    }
  } else if (wid == 0) {
    unsigned long long removed = 0ull;   // lane l holds word l
    for (int u = 0; u < na; ++u) {
      unsigned long long word = __shfl_sync(FULL, removed, u >> 6);
      if (!((word >> (u & 63)) & 1ull)) {
        if (lane == 0) keep[sorted[u]] = 1;
        if (lane < nwords) removed |= mask[u * words + lane];
      }
    }
  }
  __syncthreads();
  return na;
}

// Block-wide ordered compaction helper: exclusive prefix of 0/1 flags over
// n items processed in chunks of blockDim. pos[i] receives the rank of item i
// among flagged items; returns the total. All threads must call.
template <typename FlagFn>
__device__ int block_rank(int n, FlagFn flag, int16_t* pos, int* sh_warp /* [33] */) {
  const int tid = threadIdx.x, nt = blockDim.x, lane = lane_id(), wid = warp_id(), nw = n_warps();
  int base = 0;
  for (int c = 0; c < n; c += nt) {
    int i = c + tid;
    bool f = (i < n) && flag(i);
    unsigned b = __ballot_sync(FULL, f);
    if (lane == 0) sh_warp[wid] = __popc(b);
    __syncthreads();
    if (wid == 0) {
      int v = lane < nw ? sh_warp[lane] : 0;
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane < nw) sh_warp[lane] = incl - v;
      if (lane == 31) sh_warp[32] = incl;
    }
    __syncthreads();
    if (i < n) pos[i] = f ? static_cast<int16_t>(base + sh_warp[wid] + __popc(b & ((1u << lane) - 1u))) : -1;
    base += sh_warp[32];
    __syncthreads();
  }
  return base;
}

// Block-wide exclusive scan of one 64-bit word per thread (callers pack four
// 16-bit counters into it, so four ranks cost one scan). Returns the exclusive
// prefix; *total gets the block total. All threads must call; `sh` [33] may be
// reused only after another barrier.
__device__ inline unsigned long long block_exscan_u64(unsigned long long v, unsigned long long* sh,
                                                     unsigned long long* total) {
  const int lane = lane_id(), wid = warp_id(), nw = n_warps();
  unsigned long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sh[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const unsigned long long x = lane < nw ? sh[lane] : 0ull;
    unsigned long long xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(FULL, xi, o);
      if (lane >= o) xi += t;
    }
    if (lane < nw) sh[lane] = xi - x;
    if (lane == 31) sh[32] = xi;
  }
  __syncthreads();
  *total = sh[32];
  return sh[wid] + incl - v;
}

// ---------------------------------------------------------------- warp LAP
// Exact restatement of the solver behind hungarian_solve (tf/assoc.py:60-87 ->
// scipy.optimize.linear_sum_assignment, Crouse's shortest augmenting path; see
// oracle/lap.py) on the sentinel-padded n x n matrix, executed by ONE warp.
// Each Dijkstra iteration scans the live columns lane-parallel and reduces the
// minimum with scipy's tie rule (a free column wins; among equals the later
// list position for free columns, the earlier one otherwise), so the returned
// optimum is the one the reference gets, ties included.
//
// Row r < nr has its finite entries given by a row accessor `R` (global CSR or
// a connected component's submatrix, see CsrRows / ComponentRows); every other
// cell (including rows >= nr and columns >= nc) costs `sentinel`.
struct LapScratch {
  double *u, *v, *dist, *crow;
  int16_t *path, *row4col, *col4row, *rem, *vrows, *vcols;
};

// Finite entries of row r of the full gated matrix (CSR by row).
struct CsrRows {
  const int* rowptr;
  const int16_t* ecol;
  const double* eval;
  __device__ __forceinline__ int begin(int r) const { return rowptr[r]; }
  __device__ __forceinline__ int end(int r) const { return rowptr[r + 1]; }
  __device__ __forceinline__ int col(int e) const { return ecol[e]; }
  __device__ __forceinline__ double val(int e) const { return eval[e]; }
};

// Finite entries of local row r of one connected component: local rows map to
// global rows (ascending), global columns map to local columns.
struct ComponentRows {
  const int* rowptr;
  const int16_t* ecol;
  const double* eval;
  const int16_t* rows;     // local row -> global row
  const int16_t* colmap;   // global column -> local column
  __device__ __forceinline__ int begin(int r) const { return rowptr[rows[r]]; }
  __device__ __forceinline__ int end(int r) const { return rowptr[rows[r] + 1]; }
  __device__ __forceinline__ int col(int e) const { return colmap[ecol[e]]; }
  __device__ __forceinline__ double val(int e) const { return eval[e]; }
};

// Finite entries of local row i = one column of a connected component, when
// the component is solved transposed (columns as rows): led lists edge ids
// grouped by local row, rowmap maps a track row to its local column.
struct TransposedRows {
  const int* lrp;
  const int16_t* led;
  const int16_t* erow;
  const double* eval;
  const int16_t* rowmap;
  __device__ __forceinline__ int begin(int r) const { return lrp[r]; }
  __device__ __forceinline__ int end(int r) const { return lrp[r + 1]; }
  __device__ __forceinline__ int col(int q) const { return rowmap[erow[led[q]]]; }
  __device__ __forceinline__ double val(int q) const { return eval[led[q]]; }
};

// n_proc: rows processed. The exact reference order needs n_proc == n; when
// the optimum is known to be unique the padding rows (>= nr) may be skipped,
// since they only ever take sentinel cells.
template <class Rows>
__device__ inline void warp_lap(int n, int nr, const Rows R, double sentinel, LapScratch s, int n_proc = -1) {
  if (n_proc < 0) n_proc = n;
  const int lane = lane_id();
  for (int j = lane; j < n; j += 32) {
    s.u[j] = 0.0;
    s.v[j] = 0.0;
    s.row4col[j] = -1;
    s.col4row[j] = -1;
    s.crow[j] = sentinel;
  }
  __syncwarp();
  for (int cur = 0; cur < n_proc; ++cur) {
    for (int p = lane; p < n; p += 32) s.rem[p] = static_cast<int16_t>(n - 1 - p);
    int live = n, row = cur, nvr = 0, nvc = 0, sink = -1;
    double min_val = 0.0;
    bool first = true;
    __syncwarp();
    while (sink < 0) {
      if (lane == 0) s.vrows[nvr] = static_cast<int16_t>(row);
      ++nvr;
      int e0 = 0, e1 = 0;
      if (row < nr) {
        e0 = R.begin(row);
        e1 = R.end(row);
        for (int e = e0 + lane; e < e1; e += 32) {
          const int c = R.col(e);
          if (c >= 0) s.crow[c] = R.val(e);
        }
      }
      __syncwarp();
      const double ur = s.u[row];
      unsigned long long best = ~0ull;
      int best_p = -1;
      bool best_free = false;
      for (int p = lane; p < live; p += 32) {
        const int j = s.rem[p];
        const double r = ((min_val + s.crow[j]) - ur) - s.v[j];
        double d;
        if (first || r < s.dist[j]) {
          s.dist[j] = r;
          s.path[j] = static_cast<int16_t>(row);
          d = r;
        } else {
          d = s.dist[j];
        }
        const unsigned long long k = dkey(d);
        const bool fr = s.row4col[j] < 0;
        if (k < best || (k == best && fr)) {
          best = k;
          best_p = p;
          best_free = fr;
        }
      }
      __syncwarp();
      if (row < nr)
        for (int e = e0 + lane; e < e1; e += 32) {
          const int c = R.col(e);
          if (c >= 0) s.crow[c] = sentinel;
        }
      // warp argmin with the tie rule
      const unsigned hi = static_cast<unsigned>(best >> 32), lo = static_cast<unsigned>(best);
      const unsigned mh = __reduce_min_sync(FULL, hi);
      const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
      const bool q = best_p >= 0 && hi == mh && lo == ml;
      const unsigned fmask = __ballot_sync(FULL, q && best_free);
      int pw;
      if (fmask)
        pw = static_cast<int>(__reduce_max_sync(FULL, (q && best_free) ? static_cast<unsigned>(best_p) : 0u));
      else
        pw = static_cast<int>(__reduce_min_sync(FULL, q ? static_cast<unsigned>(best_p) : 0xffffffffu));
      const int j = s.rem[pw];
      min_val = s.dist[j];
      if (lane == 0) s.vcols[nvc] = static_cast<int16_t>(j);
      ++nvc;
      const int owner = s.row4col[j];
      if (owner < 0) sink = j; else row = owner;
      __syncwarp();
      if (lane == 0) s.rem[pw] = s.rem[live - 1];
      --live;
      first = false;
      __syncwarp();
    }
    // dual update (scipy order: u[cur] first, then visited rows / columns)
    if (lane == 0) s.u[cur] = s.u[cur] + min_val;
    for (int q = lane + 1; q < nvr; q += 32) {
      int r = s.vrows[q];
      s.u[r] = s.u[r] + (min_val - s.dist[s.col4row[r]]);
    }
    for (int q = lane; q < nvc; q += 32) {
      int j = s.vcols[q];
      s.v[j] = s.v[j] - (min_val - s.dist[j]);
    }
    __syncwarp();
    if (lane == 0) {
      int j = sink;
      while (true) {
        int i = s.path[j];
        s.row4col[j] = static_cast<int16_t>(i);
        int t = s.col4row[i];
        s.col4row[i] = static_cast<int16_t>(j);
        j = t;
        if (i == cur) break;
      }
    }
    __syncwarp();
  }
}

// Register-resident variant of warp_lap: lane l owns columns l + 32q (q < RC)
// and keeps their dual, tentative distance, path, owner and position in the
// candidate list in registers, so a Dijkstra iteration touches shared memory
// only for the current row's costs. The tie rule is applied order-free: among
// equal minima a free column with the largest list position wins, otherwise
// the smallest position (what scipy's sequential scan yields). Results land
// in s.col4row (row -> column).
template <int RC, class Rows>
__device__ inline void warp_lap_reg(int n, int nr, const Rows R, double sentinel, LapScratch s, int n_proc) {
  const int lane = lane_id();
  double v[RC], dist[RC];
  int path[RC], owner[RC], pos[RC];
#pragma unroll
  for (int q = 0; q < RC; ++q) {
    v[q] = 0.0;
    dist[q] = 0.0;
    path[q] = -1;
    owner[q] = -1;
  }
  for (int r = lane; r < n; r += 32) {
    s.u[r] = 0.0;
    s.col4row[r] = -1;
    s.crow[r] = sentinel;
  }
  __syncwarp();
  for (int cur = 0; cur < n_proc; ++cur) {
#pragma unroll
    for (int q = 0; q < RC; ++q) {
      const int j = lane + 32 * q;
      pos[q] = j < n ? n - 1 - j : -1;
    }
    int live = n, row = cur, sink = -1, nvr = 0;
    unsigned vis = 0u;
    double min_val = 0.0;
    bool first = true;
    while (sink < 0) {
      int e0 = 0, e1 = 0;
      if (row < nr) {
        e0 = R.begin(row);
        e1 = R.end(row);
        for (int e = e0 + lane; e < e1; e += 32) {
          const int c = R.col(e);
          if (c >= 0) s.crow[c] = R.val(e);
        }
      }
      __syncwarp();
      double crow[RC];
#pragma unroll
      for (int q = 0; q < RC; ++q) {
        const int j = lane + 32 * q;
        crow[q] = j < n ? s.crow[j] : sentinel;
      }
      const double ur = s.u[row];
      __syncwarp();
      if (row < nr)
        for (int e = e0 + lane; e < e1; e += 32) {
          const int c = R.col(e);
          if (c >= 0) s.crow[c] = sentinel;
        }
      unsigned long long best = ~0ull;
      int best_p = -1, best_q = 0;
      bool best_free = false;
#pragma unroll
      for (int q = 0; q < RC; ++q) {
        if (pos[q] < 0) continue;
        const double r = ((min_val + crow[q]) - ur) - v[q];
        if (first || r < dist[q]) {
          dist[q] = r;
          path[q] = row;
        }
        const unsigned long long k = dkey(dist[q]);
        const bool fr = owner[q] < 0;
        const int p = pos[q];
        bool take;
        if (best_p < 0 || k < best) take = true;
        else if (k > best) take = false;
        else take = fr ? (!best_free || p > best_p) : (!best_free && p < best_p);
        if (take) {
          best = k;
          best_p = p;
          best_q = q;
          best_free = fr;
        }
      }
      const unsigned hi = static_cast<unsigned>(best >> 32), lo = static_cast<unsigned>(best);
      const unsigned mh = __reduce_min_sync(FULL, hi);
      const unsigned ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xffffffffu);
      const bool qual = best_p >= 0 && hi == mh && lo == ml;
      const unsigned fmask = __ballot_sync(FULL, qual && best_free);
      int pw;
      if (fmask)
        pw = static_cast<int>(__reduce_max_sync(FULL, (qual && best_free) ? static_cast<unsigned>(best_p) : 0u));
      else
        pw = static_cast<int>(__reduce_min_sync(FULL, qual ? static_cast<unsigned>(best_p) : 0xffffffffu));
      const int wlane = __ffs(__ballot_sync(FULL, best_p == pw)) - 1;
      double my_d = 0.0;
      int my_o = -1;
#pragma unroll
      for (int q = 0; q < RC; ++q)
        if (q == best_q) {
          my_d = dist[q];
          my_o = owner[q];
        }
      const int q_w = __shfl_sync(FULL, best_q, wlane);
      const int j = wlane + 32 * q_w;
      min_val = __shfl_sync(FULL, my_d, wlane);
      const int own = __shfl_sync(FULL, my_o, wlane);
      if (lane == wlane) {
#pragma unroll
        for (int q = 0; q < RC; ++q)
          if (q == q_w) {
            vis |= 1u << q;
            pos[q] = -1;
          }
      }
#pragma unroll
      for (int q = 0; q < RC; ++q)          // the last list entry moves into the freed slot
        if (pos[q] == live - 1) pos[q] = pw;
      --live;
      if (own < 0) {
        sink = j;
      } else {
        if (lane == 0) {
          s.vrows[nvr] = static_cast<int16_t>(own);
          s.dist[nvr] = min_val;
        }
        ++nvr;
        row = own;
      }
      first = false;
    }
    __syncwarp();
    // dual update (scipy order: u[cur], visited rows, visited columns)
    if (lane == 0) s.u[cur] = s.u[cur] + min_val;
    for (int q2 = lane; q2 < nvr; q2 += 32) {
      const int r = s.vrows[q2];
      s.u[r] = s.u[r] + (min_val - s.dist[q2]);
    }
#pragma unroll
    for (int q = 0; q < RC; ++q)
      if ((vis >> q) & 1u) v[q] = v[q] - (min_val - dist[q]);
    __syncwarp();
    // augment along the alternating path
    int jj = sink;
    while (true) {
      const int ql = jj >> 5, ll = jj & 31;
      int pv = 0;
#pragma unroll
      for (int q = 0; q < RC; ++q)
        if (q == ql) pv = path[q];
      const int i = __shfl_sync(FULL, pv, ll);
      if (lane == ll) {
#pragma unroll
        for (int q = 0; q < RC; ++q)
          if (q == ql) owner[q] = i;
      }
      const int t = s.col4row[i];
      __syncwarp();
      if (lane == 0) s.col4row[i] = static_cast<int16_t>(jj);
      __syncwarp();
      jj = t;
      if (i == cur) break;
    }
  }
  // column duals for lap_unique (the shared-memory solver keeps them in s.v)
#pragma unroll
  for (int q = 0; q < RC; ++q) {
    const int j = lane + 32 * q;
    if (j < n) s.v[j] = v[q];
  }
  __syncwarp();
}

// Exact solver dispatch: register-resident for n <= 256, shared-memory otherwise.
template <class Rows>
__device__ inline void warp_lap_fast(int n, int nr, const Rows R, double sentinel, LapScratch s, int n_proc = -1) {
  if (n_proc < 0) n_proc = n;
  if (n <= 32) warp_lap_reg<1>(n, nr, R, sentinel, s, n_proc);
  else if (n <= 64) warp_lap_reg<2>(n, nr, R, sentinel, s, n_proc);
  else if (n <= 128) warp_lap_reg<4>(n, nr, R, sentinel, s, n_proc);
  else if (n <= 256) warp_lap_reg<8>(n, nr, R, sentinel, s, n_proc);
  else warp_lap(n, nr, R, sentinel, s, n_proc);
}

// ---------------------------------------------------------------- uniqueness
// Is the optimum just found by warp_lap on a component (rows 0..nr-1 all
// processed, columns 0..nc-1, every non-entry cell = sentinel) the only one,
// with a margin? Decides whether the component solve may stand for the
// reference's solve of the whole padded matrix: with a unique optimum (no
// other matching of the component's finite edges within eps of its cost)
// scipy, whose roundoff is far below eps, returns the same finite pairs
// whatever its processing order. Equal costs alone do not decide it either
// way (a 2 x 2 component with a + d == b + c and four distinct costs has two
// optima, while equal costs on edges that never compete leave the optimum
// unique), so the test runs on the solver's duals:
//
// with reduced costs r = c - u_i - v_j >= 0 (tight on the matching), any
// other row-perfect matching M' costs sum_{M'} r more, plus -v_c0 when it
// frees the matched column c0 of its start row (v <= 0, and 0 on free
// columns). So near-optima are exactly the alternating cycles / paths of
// cells with r <= eps, paths to a free column starting at a row whose column
// has v >= -eps. Directed graph on rows: i -> mate(j) for every cell (i, j),
// j != col(i), with r <= eps (sentinel cells too: r = sentinel - u_i - v_j,
// which never holds for an entry cell since r >= 0), i -> FREE when j is
// unmatched. An alternative changes the FINITE pairs (what the reference
// reports) iff it uses an entry cell or moves a row matched by an entry
// cell; cycles / paths made of sentinel cells only just permute padding.
// Rows with no near-tight cell can neither move nor be displaced along an
// alternative (a displaced row needs a cell of its own), so only the
// "active" rows form the graph; it is solved by one warp with a lane per
// active row (up to 32 of them, any component size; more active rows than
// that return false and the caller solves the whole padded matrix in the
// reference's order). A sentinel cell can be near-tight only for a row with
// u >= sentinel - eps (v <= 0), and never on an entry (dual feasibility).
template <class Rows>
__device__ inline void lap_row_arcs(int i, int nc, const Rows R, double sentinel, double eps, LapScratch s,
                                    const int16_t* act, unsigned& A, unsigned& FA, bool& to_free, bool& ftofree,
                                    bool& fm) {
  const int ci = s.col4row[i];
  const double ui = s.u[i];
  A = FA = 0u;
  to_free = ftofree = fm = false;
  for (int e = R.begin(i); e < R.end(i); ++e) {
    const int j = R.col(e);
    if (j < 0 || j >= nc) continue;
    if (j == ci) {
      fm = true;
      continue;
    }
    if (R.val(e) - ui - s.v[j] <= eps) {
      const int r = s.row4col[j];
      if (r < 0) {
        to_free = ftofree = true;
      } else if (act == nullptr || act[r] >= 0) {
        const unsigned bit = act ? 1u << act[r] : 1u;
        A |= bit;
        FA |= bit;
      }
    }
  }
  if (ui >= sentinel - eps) {
    const double theta = sentinel - ui - eps;
    for (int j = 0; j < nc; ++j) {
      if (j == ci || s.v[j] < theta) continue;
      const int r = s.row4col[j];
      if (r < 0) to_free = true;
      else if (act == nullptr || act[r] >= 0) A |= act ? 1u << act[r] : 1u;
    }
  }
}

// Fast pre-check for the common case of the transposed component (rows =
// detections, their entries contiguous in R's list): one lane per ENTRY
// instead of one lane per row walking its entries, so the dependent shared
// loads of a row's entries overlap. Returns true when no row is active (the
// optimum is unique; the usual outcome), false when lap_unique must build the
// graph. Other row accessors are not pre-checked.
template <class Rows>
__device__ __forceinline__ bool lap_no_active_rows(int, int, const Rows&, double, double, const LapScratch&) {
  return false;
}
__device__ __forceinline__ bool lap_no_active_rows(int nr, int nc, const TransposedRows& R, double sentinel,
                                                   double eps, const LapScratch& s) {
  const int lane = lane_id();
  const int n_ent = R.begin(nr);
  bool active = false;
  for (int q = lane; q < n_ent; q += 32) {
    int i = 0;
    while (q >= R.begin(i + 1)) ++i;
    const int j = R.col(q);
    if (j < 0 || j >= nc || j == s.col4row[i]) continue;
    if (R.val(q) - s.u[i] - s.v[j] <= eps) active = true;
  }
  for (int i = lane; i < nr; i += 32) {
    const double ui = s.u[i];
    if (ui >= sentinel - eps) {                       // a row with possible near-tight sentinel cells
      const int ci = s.col4row[i];
      const double theta = sentinel - ui - eps;
      for (int j = 0; j < nc; ++j)
        if (j != ci && s.v[j] >= theta) active = true;
    }
  }
  return !__any_sync(FULL, active);
}

template <class Rows>
// Returns 1: unique; 0: an alternative exists; -1: undecided (more than 32
// active rows) -- the caller treats both 0 and -1 as "solve the whole matrix".
__device__ inline int lap_unique(int nr, int nc, const Rows R, double sentinel, double eps, LapScratch s) {
  if (lap_no_active_rows(nr, nc, R, sentinel, eps, s)) return 1;
  const int lane = lane_id();
  for (int j = lane; j < nc; j += 32) s.row4col[j] = -1;
  __syncwarp();
  for (int i = lane; i < nr; i += 32) {
    const int c = s.col4row[i];
    if (c >= 0 && c < nc) s.row4col[c] = static_cast<int16_t>(i);
  }
  __syncwarp();
  // active rows (a near-tight cell other than their own), numbered in row order
  int16_t* act = s.rem;            // row -> active index or -1 (free scratch after the solve)
  int16_t* row_of = s.path;        // active index -> row
  int m = 0;
  for (int i0 = 0; i0 < nr; i0 += 32) {
    const int i = i0 + lane;
    bool on = false;
    if (i < nr) {
      unsigned A, FA;
      bool tf, ftf, fm;
      lap_row_arcs(i, nc, R, sentinel, eps, s, nullptr, A, FA, tf, ftf, fm);
      on = A != 0u || tf;
    }
    const unsigned bm = __ballot_sync(FULL, on);
    if (i < nr) {
      const int k = m + __popc(bm & ((1u << lane) - 1u));
      act[i] = on && k < 32 ? static_cast<int16_t>(k) : static_cast<int16_t>(-1);
      if (on && k < 32) row_of[k] = static_cast<int16_t>(i);
    }
    m += __popc(bm);
  }
  __syncwarp();
  if (m == 0) return 1;
  if (m > 32) return -1;
  // the graph on the active rows: lane a = active row row_of[a]
  unsigned A = 0u, FA = 0u;
  bool to_free = false, ftofree = false, fm = false, freeable = false;
  if (lane < m) {
    const int i = row_of[lane];
    lap_row_arcs(i, nc, R, sentinel, eps, s, act, A, FA, to_free, ftofree, fm);
    const int ci = s.col4row[i];
    freeable = ci >= 0 && ci < nc && s.v[ci] >= -eps;
  }
  // transitive closure by doubling: Rc = active rows reachable in >= 1 arcs
  unsigned Rc = A;
  for (;;) {
    unsigned nxt = Rc;
    for (int k = 0; k < m; ++k) {
      const unsigned rk = __shfl_sync(FULL, Rc, k);
      if ((Rc >> k) & 1u) nxt |= rk;
    }
    const bool changed = nxt != Rc;
    Rc = nxt;
    if (!__any_sync(FULL, changed)) break;
  }
  const unsigned tf_rows = __ballot_sync(FULL, lane < m && to_free);
  const bool free_reach = to_free || (Rc & tf_rows) != 0u;
  // rows a path alternative may start from (their column's dual ~ 0), and
  // everything they reach
  const unsigned fr_rows = __ballot_sync(FULL, lane < m && freeable);
  unsigned RF = fr_rows;
  for (int k = 0; k < m; ++k) {
    const unsigned rk = __shfl_sync(FULL, Rc, k);
    if ((fr_rows >> k) & 1u) RF |= rk;
  }
  const bool from_start = (RF >> lane) & 1u;
  const unsigned fr_reach = __ballot_sync(FULL, lane < m && free_reach);
  bool alt = false;
  if (lane < m) {
    if (fm && ((Rc >> lane) & 1u)) alt = true;                  // entry-matched row on a cycle
    if (fm && from_start && free_reach) alt = true;             // ... on a path to a free column
    if (ftofree && from_start) alt = true;                      // entry cell to a free column
  }
  // entry arcs lane -> k on a cycle (k reaches lane) or on a path (k reaches FREE)
  for (int k = 0; k < m; ++k) {
    const unsigned rk = __shfl_sync(FULL, Rc, k);
    if (lane < m && ((FA >> k) & 1u)) {
      if ((rk >> lane) & 1u) alt = true;
      if (from_start && ((fr_reach >> k) & 1u)) alt = true;
    }
  }
  return __any_sync(FULL, alt) ? 0 : 1;
}

}  // namespace tfd

