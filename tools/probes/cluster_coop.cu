// Probe (dev tool): (1) can a cooperative launch carry a cluster dimension on
// this driver; (2) cost of one "step" of a 4-CTA cluster exchanging 64 FP64
// values through distributed shared memory + a cluster barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(1, 1, 1) dummy() {}

__global__ void probe(long long* out, int steps) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  double* ring = sm;  // [2][64]
  if (threadIdx.x < 128) ring[threadIdx.x] = 0.0;
  cl.sync();
  long long t0 = clock64();
  double acc = 0.0;
  for (int s = 0; s < steps; ++s) {
    const int slot = s & 1;
    // each CTA produces 16 values and pushes them to all CTAs of the cluster
    if (threadIdx.x < 16) {
      const double v = ring[slot * 64 + ((threadIdx.x + 17) & 63)] + 1.0;
      for (unsigned r = 0; r < cl.num_blocks(); ++r) {
        double* dst = cl.map_shared_rank(ring, r);
        dst[(slot ^ 1) * 64 + rank * 16 + threadIdx.x] = v;
      }
    }
    cl.sync();
    acc += ring[(slot ^ 1) * 64 + (threadIdx.x & 63)];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x < 8) out[blockIdx.x] = (t1 - t0) / steps;
  if (acc == -1.0) out[0] = 0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 64 * sizeof(long long));
  for (int csz : {2, 4, 8}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148 / csz * csz);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = 128 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csz;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeCooperative;
    at[1].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int steps = 10000;
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe, d, steps);
    cudaError_t e2 = cudaDeviceSynchronize();
    long long h[8] = {};
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (void*)probe, &cfg);
    printf("cluster %d: coop+cluster launch: %s / %s; cycles per exchange step: %lld %lld; max active clusters %d\n",
           csz, cudaGetErrorString(e), cudaGetErrorString(e2), h[0], h[1], ncl);
  }
  return 0;
}
