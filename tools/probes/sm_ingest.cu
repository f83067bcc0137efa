// Probe (dev tool): how many bytes per SM cycle one CTA can pull from an
// L2-resident buffer -- (a) LDG.128 (.nc, no L1 allocate) into registers,
// (b) 1-D bulk async copies (TMA) into a shared-memory ring -- for 1, 8 and
// 148 CTAs.  Sizes the K^{-1} chain: its head ingests one 32 KB tile per step.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 ldg_nc(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

__global__ void __launch_bounds__(512, 1) ldg_kernel(const double2* buf, long long n_per_cta, int reps,
                                                     long long* cycles, double* sink) {
  const double2* p = buf + (long long)blockIdx.x * n_per_cta;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    for (long long i = threadIdx.x; i + 3 * 512 < n_per_cta; i += 4 * 512) {
      const double2 a = ldg_nc(p + i), b = ldg_nc(p + i + 512), c = ldg_nc(p + i + 1024), d = ldg_nc(p + i + 1536);
      acc0 += a.x + a.y;
      acc1 += b.x + b.y;
      acc2 += c.x + c.y;
      acc3 += d.x + d.y;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc0 + acc1 + acc2 + acc3 == -1.0) sink[0] = 1.0;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(128, 1) tma_kernel(const double* buf, long long bytes_per_cta, int reps,
                                                     long long* cycles) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int kStages = 4;
  constexpr unsigned kChunk = 32768;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(smem + kStages * kChunk);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const char* src = reinterpret_cast<const char*>(buf) + (long long)blockIdx.x * bytes_per_cta;
  const long long nchunks = bytes_per_cta / kChunk;
  const long long total = nchunks * reps;
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (long long g = 0; g < total + kStages; ++g) {
      if (g >= kStages) {  // wait for chunk g - kStages
        const long long w = g - kStages;
        const int s = (int)(w % kStages);
        const unsigned par = (unsigned)((w / kStages) & 1);
        unsigned ok = 0;
        while (!ok)
          asm volatile(
              "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n}"
              : "=r"(ok)
              : "r"(smem_u32(bar + s)), "r"(par)
              : "memory");
      }
      if (g < total) {
        const int s = (int)(g % kStages);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar + s)), "r"(kChunk)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(smem + (size_t)s * kChunk)),
            "l"(src + (g % nchunks) * kChunk), "r"(kChunk), "r"(smem_u32(bar + s))
            : "memory");
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  const long long per_cta = 2ll << 20;  // 2 MB per CTA
  const int maxg = 148;
  double* buf;
  cudaMalloc(&buf, per_cta * maxg);
  cudaMemset(buf, 0, per_cta * maxg);
  long long* cyc;
  double* sink;
  cudaMalloc(&cyc, maxg * sizeof(long long));
  cudaMalloc(&sink, 8);
  long long h[maxg];
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * 32768 + 64);
  for (int grid : {1, 8, 32, 148}) {
    const int reps = 20;
    // L2 residency: 148 x 2 MB exceeds L2, so the 148-CTA rows are HBM-bound
    ldg_kernel<<<grid, 512>>>((const double2*)buf, per_cta / 16, 1, cyc, sink);
    ldg_kernel<<<grid, 512>>>((const double2*)buf, per_cta / 16, reps, cyc, sink);
    cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("LDG.128  grid %3d: %.1f B/cycle/SM (%.0f cycles for %lld B)\n", grid, per_cta * reps / mx, mx,
           per_cta * reps);
    tma_kernel<<<grid, 128, 4 * 32768 + 64>>>(buf, per_cta, 1, cyc);
    tma_kernel<<<grid, 128, 4 * 32768 + 64>>>(buf, per_cta, reps, cyc);
    cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("TMA bulk grid %3d: %.1f B/cycle/SM\n", grid, per_cta * reps / mx);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
