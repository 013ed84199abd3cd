// DSMEM / proxy-fence / bulk-copy latency micro-benchmarks on B200 (cluster of 8).
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__global__ void __cluster_dims__(8, 1, 1) k(long long* out, const float* g, int n) {
  __shared__ int buf[1024];
  __shared__ __align__(16) float stage[4096];
  __shared__ unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = (i * 7 + 1) & 1023;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  long long r[8] = {0};
  if (rank == 1 && threadIdx.x == 0) {
    int* rb = cl.map_shared_rank(buf, 0);
    int p = 0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) p = rb[p];                 // generic-pointer DSMEM dependent chain
    long long t1 = clock64();
    r[0] = (t1 - t0) / n; r[7] += p;
    unsigned base = su32(buf), rbase;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(rbase) : "r"(base));
    p = 0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) {
      int v;
      asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(rbase + 4 * p));
      p = v;
    }
    t1 = clock64();
    r[1] = (t1 - t0) / n; r[7] += p;
    t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("fence.proxy.async;" ::: "memory");
    t1 = clock64();
    r[2] = (t1 - t0) / n;
    t0 = clock64();
    for (int i = 0; i < n; ++i) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    t1 = clock64();
    r[3] = (t1 - t0) / n;
    // bulk copy 2 KB global -> smem, round trip
    unsigned ph = 0;
    t0 = clock64();
    for (int i = 0; i < n / 16; ++i) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(2048) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(stage)), "l"(g + (i % 64) * 512), "r"(2048), "r"(su32(&bar)) : "memory");
      asm volatile("{ .reg .pred p; W_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W_%=; }"
                   ::"r"(su32(&bar)), "r"(ph) : "memory");
      ph ^= 1;
    }
    t1 = clock64();
    r[4] = (t1 - t0) / (n / 16);
    // global load latency (L2 hit), dependent
    const int* gi = reinterpret_cast<const int*>(g);
    p = 0;
    t0 = clock64();
    for (int i = 0; i < n; ++i) p = __ldcg(gi + (p & 4095)) & 4095;
    t1 = clock64();
    r[5] = (t1 - t0) / n; r[7] += p;
    // remote store throughput (fire and forget)
    t0 = clock64();
    for (int i = 0; i < n; ++i) rb[i & 1023] = i;
    t1 = clock64();
    r[6] = (t1 - t0) / n;
    for (int i = 0; i < 8; ++i) out[i] = r[i];
  }
  cl.sync();
  // contention: all 7 followers x 256 threads hammer rank 0 with generic loads of the same address
  long long t0 = clock64();
  int acc = 0;
  if (rank != 0) {
    int* rb = cl.map_shared_rank(buf, 0);
    for (int i = 0; i < 16; ++i) acc += rb[(acc + i) & 7];
  }
  long long t1 = clock64();
  if (rank == 1 && threadIdx.x == 0) { out[8] = (t1 - t0) / 16; out[9] = acc; }
  cl.sync();
  t0 = clock64();
  acc = 0;
  if (rank != 0 && (threadIdx.x & 31) == 0) {
    int* rb = cl.map_shared_rank(buf, 0);
    for (int i = 0; i < 16; ++i) acc += rb[(acc + i) & 7];
  }
  t1 = clock64();
  if (rank == 1 && threadIdx.x == 0) { out[10] = (t1 - t0) / 16; out[11] = acc; }
}
int main() {
  long long* o; float* g;
  cudaMallocManaged(&o, 16 * sizeof(long long));
  cudaMalloc(&g, 64 * 2048);
  cudaMemset(g, 0, 64 * 2048);
  k<<<8, 256>>>(o, g, 256);
  k<<<8, 256>>>(o, g, 256);
  cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  const char* names[] = {"dsmem generic ld (dep)", "ld.shared::cluster (dep)", "fence.proxy.async", "fence.proxy.async.shared::cta",
                         "bulk 2KB g->s round trip", "ld.global.cg L2 hit (dep)", "dsmem generic st (issue)", "-",
                         "all-thread generic ld x7 CTAs (per ld)", "-", "lane0-only generic ld x7 CTAs (per ld)"};
  for (int i = 0; i < 11; ++i) if (names[i][0] != '-') printf("%-42s %lld cycles\n", names[i], o[i]);
}
