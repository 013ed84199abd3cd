// Micro-benchmark of the association's cost phase pattern at config-4 shape:
// G CTAs (one per stream, 2 per SM), each runs F frames of E fp64 dot products
// between random pairs of its track-pool rows and that frame's detection rows
// (512-d). Variants: 0 = fp32 rows, F2F to fp64 + DFMA (today);
// 1 = fp64 rows (values exact in fp32), DFMA only; 2 = fp32 rows, integer
// fp32 -> fp64 conversion (exact for normal numbers / zero) + DFMA;
// 3 = fp32 rows, fp32 FMA (wrong numerics, timing bound only).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a costbw.cu -o costbw
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int D = 512, TR = 112, KD = 48, F = 8, E = 340;

__device__ __forceinline__ double cvt_int(float f) {
  const unsigned x = __float_as_uint(f);
  const unsigned ax = x & 0x7fffffffu;
  unsigned hi = ((ax >> 3) + 0x38000000u) | (x & 0x80000000u);
  hi = ax ? hi : (x & 0x80000000u);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(x << 29));
}

template <int V, int NB>
__global__ void __launch_bounds__(128, 2) cost_kernel(const float* pool32, const double* pool64, const float* det32,
                                                      const double* det64, const short2* pairs, double* out) {
  const int g = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double sink = 0.0;
  for (int f = 0; f < F; ++f) {
    const short2* pr = pairs + (static_cast<long long>(g) * F + f) * E;
    const long long pbase = static_cast<long long>(g) * TR * D;
    const long long dbase = (static_cast<long long>(g) * F + f) * KD * D;
    for (int e0 = NB * w; e0 < E; e0 += NB * nw) {
      double acc[NB];
      int t[NB], k[NB];
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const short2 p = pr[min(e0 + j, E - 1)];
        t[j] = p.x;
        k[j] = p.y;
        acc[j] = 0.0;
      }
      if (V == 1) {
        double2 a[NB][4], b[NB][4];
#pragma unroll
        for (int j = 0; j < NB; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a[j][q] = reinterpret_cast<const double2*>(pool64 + pbase + t[j] * D)[lane + 32 * q];
            b[j][q] = reinterpret_cast<const double2*>(det64 + dbase + k[j] * D)[lane + 32 * q];
          }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            acc[j] = fma(a[j][q].x, b[j][q].x, acc[j]);
            acc[j] = fma(a[j][q].y, b[j][q].y, acc[j]);
          }
#pragma unroll
        for (int j = 0; j < NB; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a[j][q] = reinterpret_cast<const double2*>(pool64 + pbase + t[j] * D)[128 + lane + 32 * q];
            b[j][q] = reinterpret_cast<const double2*>(det64 + dbase + k[j] * D)[128 + lane + 32 * q];
          }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
          for (int j = 0; j < NB; ++j) {
            acc[j] = fma(a[j][q].x, b[j][q].x, acc[j]);
            acc[j] = fma(a[j][q].y, b[j][q].y, acc[j]);
          }
      } else {
        float4 a[NB][4], b[NB][4];
#pragma unroll
        for (int j = 0; j < NB; ++j)
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            a[j][q] = reinterpret_cast<const float4*>(pool32 + pbase + t[j] * D)[lane + 32 * q];
            b[j][q] = reinterpret_cast<const float4*>(det32 + dbase + k[j] * D)[lane + 32 * q];
          }
        if (V == 4) {
          // double-float: exact fp32 products (p + e), TwoSum accumulation of p, e summed plainly
          float sh[NB], sl[NB];
#pragma unroll
          for (int j = 0; j < NB; ++j) { sh[j] = 0.f; sl[j] = 0.f; }
#define DF_TERM(X, Y)                                   \
  {                                                     \
    const float p_ = __fmul_rn(X, Y);                   \
    const float e_ = __fmaf_rn(X, Y, -p_);              \
    const float t_ = __fadd_rn(sh[j], p_);              \
    const float z_ = __fsub_rn(t_, sh[j]);              \
    const float r_ = __fadd_rn(__fsub_rn(sh[j], __fsub_rn(t_, z_)), __fsub_rn(p_, z_)); \
    sl[j] = __fadd_rn(sl[j], __fadd_rn(r_, e_));        \
    sh[j] = t_;                                         \
  }
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < NB; ++j) {
              DF_TERM(a[j][q].x, b[j][q].x)
              DF_TERM(a[j][q].y, b[j][q].y)
              DF_TERM(a[j][q].z, b[j][q].z)
              DF_TERM(a[j][q].w, b[j][q].w)
            }
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[j] = (double)sh[j] + (double)sl[j];
        } else if (V == 3) {
          float af[NB];
#pragma unroll
          for (int j = 0; j < NB; ++j) af[j] = 0.f;
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < NB; ++j) {
              af[j] = fmaf(a[j][q].x, b[j][q].x, af[j]);
              af[j] = fmaf(a[j][q].y, b[j][q].y, af[j]);
              af[j] = fmaf(a[j][q].z, b[j][q].z, af[j]);
              af[j] = fmaf(a[j][q].w, b[j][q].w, af[j]);
            }
#pragma unroll
          for (int j = 0; j < NB; ++j) acc[j] = af[j];
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int j = 0; j < NB; ++j) {
              if (V == 0) {
                acc[j] = fma((double)a[j][q].x, (double)b[j][q].x, acc[j]);
                acc[j] = fma((double)a[j][q].y, (double)b[j][q].y, acc[j]);
                acc[j] = fma((double)a[j][q].z, (double)b[j][q].z, acc[j]);
                acc[j] = fma((double)a[j][q].w, (double)b[j][q].w, acc[j]);
              } else {
                acc[j] = fma(cvt_int(a[j][q].x), cvt_int(b[j][q].x), acc[j]);
                acc[j] = fma(cvt_int(a[j][q].y), cvt_int(b[j][q].y), acc[j]);
                acc[j] = fma(cvt_int(a[j][q].z), cvt_int(b[j][q].z), acc[j]);
                acc[j] = fma(cvt_int(a[j][q].w), cvt_int(b[j][q].w), acc[j]);
              }
            }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int j = 0; j < NB; ++j) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
#pragma unroll
      for (int j = 0; j < NB; ++j) sink += acc[j];
    }
    __syncthreads();
  }
  if (lane == 0) out[g * nw + w] = sink;
}

template <int V, int NB>
float run(int G, const float* p32, const double* p64, const float* d32, const double* d64, const short2* pr, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cost_kernel<V, NB><<<G, 128>>>(p32, p64, d32, d64, pr, out);
  cudaEventRecord(e0);
  for (int i = 0; i < 5; ++i) cost_kernel<V, NB><<<G, 128>>>(p32, p64, d32, d64, pr, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main(int argc, char** argv) {
  const int G = argc > 1 ? atoi(argv[1]) : 296;
  const size_t np = (size_t)G * TR * D, nd = (size_t)G * F * KD * D, npr = (size_t)G * F * E;
  std::vector<float> hp(np), hd(nd);
  for (auto& x : hp) x = (rand() / (float)RAND_MAX - 0.5f) * 0.08f;
  for (auto& x : hd) x = (rand() / (float)RAND_MAX - 0.5f) * 0.08f;
  std::vector<double> hp64(hp.begin(), hp.end()), hd64(hd.begin(), hd.end());
  std::vector<short2> hpr(npr);
  const bool csr = argc > 2;   // CSR-like order: entries grouped by track (~3 per track), as the kernel sees them
  for (size_t i = 0; i < npr; ++i) {
    const int e = i % E;
    hpr[i] = csr ? make_short2((e * TR) / E, rand() % KD) : make_short2(rand() % TR, rand() % KD);
  }
  float *p32, *d32;
  double *p64, *d64, *out;
  short2* pr;
  cudaMalloc(&p32, np * 4); cudaMalloc(&d32, nd * 4); cudaMalloc(&p64, np * 8); cudaMalloc(&d64, nd * 8);
  cudaMalloc(&pr, npr * 4); cudaMalloc(&out, G * 64 * 8);
  cudaMemcpy(p32, hp.data(), np * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d32, hd.data(), nd * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(p64, hp64.data(), np * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(d64, hd64.data(), nd * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(pr, hpr.data(), npr * 4, cudaMemcpyHostToDevice);
  // check variant 2 conversion equals the hardware one on the data
  const char* names[] = {"fp32 rows + F2F + DFMA", "fp64 rows + DFMA", "fp32 rows + int cvt + DFMA", "fp32 FMA (timing only)", "double-float fp32 (no F2F)"};
  float t[5][3];
  t[0][0] = run<0, 2>(G, p32, p64, d32, d64, pr, out); t[0][1] = run<0, 4>(G, p32, p64, d32, d64, pr, out);
  t[1][0] = run<1, 2>(G, p32, p64, d32, d64, pr, out); t[1][1] = run<1, 4>(G, p32, p64, d32, d64, pr, out);
  t[2][0] = run<2, 2>(G, p32, p64, d32, d64, pr, out); t[2][1] = run<2, 4>(G, p32, p64, d32, d64, pr, out);
  t[3][0] = run<3, 2>(G, p32, p64, d32, d64, pr, out); t[3][1] = run<3, 4>(G, p32, p64, d32, d64, pr, out);
  t[4][0] = run<4, 2>(G, p32, p64, d32, d64, pr, out); t[4][1] = run<4, 4>(G, p32, p64, d32, d64, pr, out);
  for (int v = 0; v < 5; ++v)
    printf("G=%d %-28s NB=2: %.1f us/launch (%.2f us/frame)  NB=4: %.1f us/launch (%.2f us/frame)\n", G, names[v],
           t[v][0] * 1e3, t[v][0] * 1e3 / F, t[v][1] * 1e3, t[v][1] * 1e3 / F);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
