// Exhaustive-ish check of div_by (Markstein division from __drcp_rn) against
// IEEE division on random and adversarial operands in the ranges the kernels
// use it for (embedding components / fp64 norms).
#include <cstdio>
#include <cstdint>
#include "../../paper_2011_03910_b200/csrc/tf_device.cuh"
using namespace tfd;
__device__ unsigned long long xorshift(unsigned long long& s) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
__global__ void check(unsigned long long seed, long long iters, unsigned long long* bad, unsigned long long* bad32) {
  unsigned long long s = seed ^ (0x9E3779B97F4A7C15ull * (blockIdx.x * blockDim.x + threadIdx.x + 1));
  unsigned long long nb = 0, nb32 = 0;
  for (long long i = 0; i < iters; ++i) {
    const unsigned long long r1 = xorshift(s), r2 = xorshift(s);
    // a: random sign/exponent in [2^-30, 2^4), full mantissa; b: [2^-10, 2^20)
    const double a = __longlong_as_double(static_cast<long long>((r1 & 0x800FFFFFFFFFFFFFull) |
                                                                  (static_cast<unsigned long long>(1023 - 30 + (r1 >> 52) % 34) << 52)));
    const double b = __longlong_as_double(static_cast<long long>((r2 & 0x000FFFFFFFFFFFFFull) |
                                                                  (static_cast<unsigned long long>(1023 - 10 + (r2 >> 52) % 30) << 52)));
    const double y = __drcp_rn(b);
    const double q = div_by(a, b, y), t = a / b;
    nb += __double_as_longlong(q) != __double_as_longlong(t);
    nb32 += __float_as_int(static_cast<float>(q)) != __float_as_int(static_cast<float>(t));
  }
  atomicAdd(bad, nb);
  atomicAdd(bad32, nb32);
}
int main() {
  unsigned long long *bad, *bad32;
  cudaMallocManaged(&bad, 8); cudaMallocManaged(&bad32, 8);
  *bad = 0; *bad32 = 0;
  const int blocks = 148 * 8, threads = 256; const long long iters = 4096;
  for (int rep = 0; rep < 8; ++rep) check<<<blocks, threads>>>(1234567ull + rep, iters, bad, bad32);
  cudaDeviceSynchronize();
  printf("divisions checked: %lld, fp64 mismatches: %llu, fp32-output mismatches: %llu (%s)\n",
         8LL * blocks * threads * iters, *bad, *bad32, cudaGetErrorString(cudaGetLastError()));
  return *bad != 0;
}
