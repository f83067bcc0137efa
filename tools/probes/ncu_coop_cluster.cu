// Probe (dev tool): which cooperative + cluster launch configurations can
// ncu profile?  Variants: static smem, grid size, stream, st.async.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

struct Args { long long* out; int steps; double pad[48]; };

template <bool kStatic>
__global__ void __launch_bounds__(512, 1) probe(const Args a) {
  extern __shared__ double sm[];
  __shared__ double st[kStatic ? 5000 : 1];
  cg::cluster_group cl = cg::this_cluster();
  st[threadIdx.x % (kStatic ? 5000 : 1)] = 1.0;
  sm[threadIdx.x] = st[0];
  cl.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) a.out[0] = (long long)sm[0];
}

int main(int argc, char** argv) {
  const int variant = atoi(argv[1]);
  long long* d;
  cudaMalloc(&d, 64);
  cudaStream_t s = 0;
  if (variant & 4) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const bool stat = variant & 1;
  const int grid = (variant & 2) ? 130 : 148;
  auto fn = stat ? probe<true> : probe<false>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 131104);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = 131104;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = 2; at[1].val.clusterDim.y = 1; at[1].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = (variant & 8) ? 1 : 2;  // 8: cooperative only
  Args a{};
  a.out = d;
  a.steps = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, fn, a);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("variant %d (static=%d grid=%d stream=%d attrs=%d): %s / %s\n", variant, stat, grid, (variant & 4) != 0,
         cfg.numAttrs, cudaGetErrorString(e), cudaGetErrorString(e2));
  return e != cudaSuccess || e2 != cudaSuccess;
}
