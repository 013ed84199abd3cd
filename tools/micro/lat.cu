// Latency micro-benchmarks on B200 (clock64 per dependent chain).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__global__ void k_dadd(double* out, long long* cyc, double a, int n) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + a; x = x * a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_ddiv(double* out, long long* cyc, double a, int n) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = a / x; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_dsqrt(double* out, long long* cyc, double a, int n) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = 1.0 / sqrt(x); }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_fadd(float* out, long long* cyc, float a, int n) {
  float x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + a; x = x * a; }
  long long t1 = clock64();
  out[threadIdx.x] = x; if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}
// throughput: 8 independent chains per thread
__global__ void k_dthr(double* out, long long* cyc, double a, int n) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = a + threadIdx.x + j;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, a);
  }
  long long t1 = clock64();
  double s = 0; for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s; if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_sync(long long* cyc, int n) {
  __shared__ int s; if (threadIdx.x == 0) s = 0; __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { if (threadIdx.x == (i & 255)) s += 1; __syncthreads(); }
  int v = s;
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0); cyc[1] = v; }
}
__global__ void k_lds(long long* cyc, int n) {
  __shared__ int buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = buf[p];
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0); cyc[1] = p; }
}
__global__ void __cluster_dims__(8, 1, 1) k_csync(long long* cyc, int n) {
  cg::cluster_group cl = cg::this_cluster();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) cl.sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = (t1 - t0);
}
__global__ void k_shfl(long long* cyc, int n) {
  int v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __shfl_xor_sync(0xffffffff, v, 1) + 1;
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0); cyc[1] = v; }
}
__global__ void k_ballot(long long* cyc, int n) {
  unsigned v = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) v = __ballot_sync(0xffffffff, (v >> (threadIdx.x & 31)) & 1) + threadIdx.x;
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0); cyc[1] = v; }
}
__global__ void k_atoms(long long* cyc, int n) {
  __shared__ unsigned long long m[64];
  if (threadIdx.x < 64) m[threadIdx.x] = ~0ull; __syncthreads();
  long long t0 = clock64();
  unsigned long long r = 0;
  for (int i = 0; i < n; ++i) r += atomicMin(&m[(threadIdx.x + i) & 63], (unsigned long long)(threadIdx.x * 7 + i + r % 3));
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = (t1 - t0); cyc[1] = r; }
}
int main() {
  double* od; float* of; long long* c; cudaMalloc(&od, 1 << 22); cudaMalloc(&of, 1 << 20); cudaMallocManaged(&c, 64);
  const int n = 4096;
  auto rep = [&](const char* name, double per) { cudaDeviceSynchronize(); printf("%-34s %8.2f cycles/op\n", name, (double)c[0] / per); };
  k_dadd<<<1, 32>>>(od, c, 1.0000001, n); k_dadd<<<1, 32>>>(od, c, 1.0000001, n); rep("dadd+dmul dependent (per op)", 2.0 * n);
  k_fadd<<<1, 32>>>(of, c, 1.0000001f, n); rep("fadd+fmul dependent (per op)", 2.0 * n);
  k_ddiv<<<1, 32>>>(od, c, 1.5, n); rep("ddiv dependent", n);
  k_dsqrt<<<1, 32>>>(od, c, 1.5, n); rep("1/sqrt(double) dependent", n);
  k_dthr<<<1, 32>>>(od, c, 1.0000001, n); rep("dfma 1 warp 8 chains (per warp-op)", 8.0 * n);
  k_dthr<<<1, 128>>>(od, c, 1.0000001, n); rep("dfma 4 warps 8 chains", 8.0 * n);
  k_dthr<<<1, 256>>>(od, c, 1.0000001, n); rep("dfma 8 warps 8 chains", 8.0 * n);
  k_dthr<<<1, 1024>>>(od, c, 1.0000001, n); rep("dfma 32 warps 8 chains", 8.0 * n);
  k_sync<<<1, 256>>>(c, n); rep("syncthreads 8 warps (+sts)", n);
  k_sync<<<1, 512>>>(c, n); rep("syncthreads 16 warps (+sts)", n);
  k_sync<<<1, 1024>>>(c, n); rep("syncthreads 32 warps (+sts)", n);
  k_lds<<<1, 32>>>(c, n); rep("lds dependent", n);
  k_csync<<<8, 256>>>(c, 1024); rep("cluster.sync 8 CTAs x 256", 1024);
  k_shfl<<<1, 32>>>(c, n); rep("shfl dependent", n);
  k_ballot<<<1, 32>>>(c, n); rep("ballot dependent", n);
  k_atoms<<<1, 256>>>(c, n); rep("atoms.min.u64 dependent (8 warps)", n);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
