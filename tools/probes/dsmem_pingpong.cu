// Probe (dev tool): round-trip latency of one 8-byte hand-off between two CTAs
// of a cluster (ping-pong, 2000 round trips), by mechanism:
//   0: st.relaxed.cluster.shared::cluster  + ld.relaxed.cluster.shared::cta poll
//   1: st.shared::cluster (weak)           + ld.volatile.shared poll
//   2: st.async + mbarrier complete_tx     + mbarrier.try_wait.parity
//   3: remote poll: ld.relaxed.cluster.shared::cluster of the peer's slot
//   4: global memory: st.relaxed.gpu + ld.relaxed.gpu poll (L2)
// Sizes the K^{-1} chain's head <-> tail hand-offs.
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

__global__ void __cluster_dims__(2, 1, 1) pingpong(int mode, int iters, long long* out, unsigned long long* g) {
  __shared__ unsigned long long slot[2];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned me = blockIdx.x & 1, other = me ^ 1;
  if (threadIdx.x == 0) {
    slot[0] = slot[1] = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (blockIdx.x < 2 && threadIdx.x == 0) g[blockIdx.x] = 0;
  __syncthreads();
  csync();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    const unsigned remote_slot = mapa(&slot[0], other);
    const unsigned remote_bar = mapa(&bar, other);
    for (int it = 1; it <= iters; ++it) {
      const unsigned long long want = (unsigned long long)it;
      // CTA 0 sends first, CTA 1 answers
      if (me == 0) {
        // send it, wait for reply it
        if (mode == 0) asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(remote_slot), "l"(want) : "memory");
        if (mode == 1) asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(remote_slot), "l"(want) : "memory");
        if (mode == 2) {
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];" ::"r"(remote_slot),
                       "l"(want), "r"(remote_bar)
                       : "memory");
        }
        if (mode == 3) slot[1] = want;  // publish locally; the peer pulls
        if (mode == 4) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(g + 1), "l"(want) : "memory");
      }
      // wait for `want` (CTA 1: the ping; CTA 0: the pong)
      unsigned long long v = 0;
      if (mode == 0) {
        do asm volatile("ld.relaxed.cluster.shared::cta.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(&slot[0])) : "memory");
        while (v != want);
      } else if (mode == 1) {
        do v = *(volatile unsigned long long*)&slot[0];
        while (v != want);
      } else if (mode == 2) {
        unsigned ok = 0;
        const unsigned par = (unsigned)((it - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 8;" ::"r"(smem_u32(&bar)) : "memory");
        while (!ok)
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
              : "=r"(ok)
              : "r"(smem_u32(&bar)), "r"(par)
              : "memory");
      } else if (mode == 3) {
        const unsigned peer_pub = mapa(&slot[1], other);
        do asm volatile("ld.relaxed.cluster.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(peer_pub) : "memory");
        while (v != want);
      } else {
        do asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(g + me) : "memory");
        while (v != want);
      }
      if (me == 1) {  // reply
        if (mode == 0) asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(remote_slot), "l"(want) : "memory");
        if (mode == 1) asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(remote_slot), "l"(want) : "memory");
        if (mode == 2) {
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u64 [%0], %1, [%2];" ::"r"(remote_slot),
                       "l"(want), "r"(remote_bar)
                       : "memory");
        }
        if (mode == 3) slot[1] = want;
        if (mode == 4) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(g + 0), "l"(want) : "memory");
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && me == 0) out[mode] = (t1 - t0) / iters;
  csync();
}

int main() {
  long long* out;
  unsigned long long* g;
  cudaMalloc(&out, 8 * sizeof(long long));
  cudaMalloc(&g, 16 * sizeof(unsigned long long));
  const char* names[] = {"st.relaxed.cluster remote + local poll", "st.shared::cluster weak + volatile poll",
                         "st.async + mbarrier try_wait", "local publish + remote ld poll",
                         "global st.relaxed.gpu + ld poll (L2)"};
  for (int mode = 0; mode < 5; ++mode) {
    // mode 2's mbarrier phase bookkeeping assumes the expect_tx happens before the data: the
    // receiving side arms with its own expect_tx each round (sender arms the peer's? no: each
    // CTA arms its own barrier right after its previous wait) -- good enough for latency
    pingpong<<<2, 32>>>(mode, 2000, out, g);
    cudaError_t e = cudaDeviceSynchronize();
    long long h = 0;
    cudaMemcpy(&h, out + mode, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d (%s): %lld cycles per round trip (%s)\n", mode, names[mode], h, cudaGetErrorString(e));
  }
  return 0;
}
