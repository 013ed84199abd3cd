// Issue cost of the cluster hand-off primitives on B200, seen by the issuing
// thread (clock64): remote relaxed mbarrier arrives, st.async, bulk copies to
// a peer CTA's shared memory, fence.acq_rel.cluster, split cluster barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o handoff handoff.cu
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(const void* p, unsigned r) {
  unsigned x; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(x) : "r"(su32(p)), "r"(r)); return x;
}

__global__ void __cluster_dims__(8, 1, 1) k(long long* out, int n_peers, int mode) {
  __shared__ __align__(16) int buf[1024];
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(&bar)), "r"((1 << 20) - 1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = i;
  __syncthreads();
  cl.sync();
  if (rank == 0 && threadIdx.x == 0) {
    long long t[8];
    for (int i = 0; i < 8; ++i) t[i] = 0;
    t[0] = clock64();
    if (mode & 1) for (int r = 1; r <= n_peers; ++r)
      asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa(&bar, r)) : "memory");
    t[1] = clock64();
    if (mode & 2) for (int r = 1; r <= n_peers; ++r)
      asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" :: "r"(mapa(&bar, r)), "r"(0u) : "memory");
    t[2] = clock64();
    if (mode & 4) for (int r = 1; r <= n_peers; ++r)
      asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1,%2,%3,%4}, [%5];"
                   :: "r"(mapa(buf, r)), "r"(1), "r"(2), "r"(3), "r"(4), "r"(mapa(&bar, r)) : "memory");
    t[3] = clock64();
    if (mode & 8) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (mode & 8) for (int r = 1; r <= n_peers; ++r)
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   "cp.async.bulk.commit_group;" :: "r"(mapa(buf + 256, r)), "r"(su32(buf)), "r"(128u), "r"(mapa(&bar, r)) : "memory");
    t[4] = clock64();
    if (mode & 16) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    t[5] = clock64();
    if (mode & 32) asm volatile("fence.acq_rel.cluster;" ::: "memory");
    t[6] = clock64();
    if (mode & 64) for (int r = 1; r <= n_peers; ++r)
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(mapa(&bar, r)) : "memory");
    t[7] = clock64();
    for (int i = 0; i < 7; ++i) out[i] = t[i + 1] - t[i];
  }
  __syncthreads();
  cl.sync();
  {
    long long a = clock64();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    long long b = clock64();
    if (rank == 0 && threadIdx.x == 0) out[7] = b - a;
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main(int argc, char** argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  const int mode = argc > 1 ? atoi(argv[1]) : 127;
  long long* d; cudaMalloc(&d, 8 * sizeof(long long));
  const char* names[8] = {"relaxed remote arrive", "relaxed remote arrive.expect_tx", "st.async v4",
                          "fence.proxy.async + bulk copy 128B", "bulk wait_group.read", "fence.acq_rel.cluster",
                          "release remote arrive", "barrier.cluster.arrive.release (1 thread timed)"};
  for (int peers : {1, 7}) {
    long long h[8] = {0};
    for (int rep = 0; rep < 5; ++rep) {
      k<<<8, 32>>>(d, peers, mode);
      cudaDeviceSynchronize();
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    }
    cudaError_t e = cudaGetLastError();
    printf("mode=%d peers=%d (%s)\n", mode, peers, cudaGetErrorString(e));
    for (int i = 0; i < 8; ++i) printf("  %-48s %6lld cycles%s\n", names[i], h[i], i < 4 || i == 6 ? " total" : "");
  }
  return 0;
}
