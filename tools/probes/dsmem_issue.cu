// Probe (dev tool): issue cost of back-to-back remote shared-memory stores
// from one thread (does the warp block per store?), 8-byte values to a
// cluster peer: st.relaxed.cluster.shared::cluster, st.shared::cluster (weak),
// st.async + mbarrier complete_tx; also a local st.shared for reference.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(const void* p, unsigned r) {
  unsigned a;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(smem_u32(p)), "r"(r));
  return a;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int MODE, int N>
__global__ void __cluster_dims__(2, 1, 1) issue(long long* out) {
  __shared__ double buf[1024];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  csync();
  const unsigned me = blockIdx.x & 1;
  long long dt = 0;
  if (me == 0 && threadIdx.x < 32) {
    const unsigned rb = mapa(&buf[0], 1), rbar = mapa(&bar, 1);
    const long long t0 = clock64();
#pragma unroll
    for (int j = 0; j < N; ++j) {
      const unsigned a = rb + (unsigned)((j * 32 + threadIdx.x) % 1024) * 8u;
      const double v = (double)j;
      if (MODE == 0) asm volatile("st.relaxed.cluster.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
      if (MODE == 1) asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
      if (MODE == 2)
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(a), "d"(v),
                     "r"(rbar)
                     : "memory");
      if (MODE == 3) buf[(j * 32 + threadIdx.x) % 1024] = v;
    }
    const long long t1 = clock64();
    dt = t1 - t0;
    if (threadIdx.x == 0) out[0] = dt;
  }
  // peer: accept the st.async bytes so the barrier phase can complete
  if (MODE == 2 && me == 1 && threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(N * 32 * 8)
                 : "memory");
  __syncthreads();
  csync();
}

template <int MODE, int N>
void run(const char* name, long long* d) {
  issue<MODE, N><<<2, 64>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-36s N=%2d: %5lld cycles issue (%.1f per store) %s\n", name, N, h, (double)h / N, cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 64);
  run<0, 1>("st.relaxed.cluster.shared::cluster", d);
  run<0, 8>("st.relaxed.cluster.shared::cluster", d);
  run<0, 32>("st.relaxed.cluster.shared::cluster", d);
  run<1, 1>("st.shared::cluster (weak)", d);
  run<1, 8>("st.shared::cluster (weak)", d);
  run<1, 32>("st.shared::cluster (weak)", d);
  run<2, 1>("st.async + complete_tx", d);
  run<2, 8>("st.async + complete_tx", d);
  run<2, 32>("st.async + complete_tx", d);
  run<3, 8>("local st.shared", d);
  run<3, 32>("local st.shared", d);
  return 0;
}
