// Probe: latency of a grid-level blocked chain step for the K^{-1} sweeps
// with explicit super-block inverses.  C CTAs each own R = 512 / C rows of
// y_S = A_S [c_S; y_{S-1}] (a dense 512 x 1024 matvec per step, operands
// resident in shared memory), publish their R values to global slots armed
// with a NaN sentinel, and every CTA polls all 512 values of the previous
// step before the next.  Prints the time per step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/probes/superchain.cu -o tools/probes/superchain
#include <cstdio>
#include <vector>

constexpr int kN = 512;          // rows per super step
constexpr int kK = 2 * kN;       // [c_S; y_{S-1}]
constexpr unsigned long long kSent = ~0ull;

__device__ __forceinline__ unsigned long long ldr(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int R>
__global__ void __launch_bounds__(512, 1) superchain(double* ybuf, const double* A, int steps, long long* cyc) {
  extern __shared__ double sm[];
  double* As = sm;              // [R][kK]
  double* yv = sm + R * kK;     // [kK]
  __shared__ double part[R][16];
  const int tid = threadIdx.x;
  for (int e = tid; e < R * kK; e += 512) As[e] = A[(size_t)blockIdx.x * R * kK + e];
  __syncthreads();
  constexpr int TPR = 512 / R;   // threads per row
  constexpr int PER = kK / TPR;  // products per thread
  const int row = tid / TPR, sub = tid % TPR;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    // c_S (pretend the workers' hand-off is ready) and y_{S-1} from every CTA
    yv[tid] = 1.0 / (1 + tid);
    const double* src = ybuf + (size_t)s * kN + tid;
    unsigned long long v = ldr(src);
    while (v == kSent) v = ldr(src);
    yv[kN + tid] = __longlong_as_double((long long)v);
    __syncthreads();
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < PER; ++q) acc = fma(As[row * kK + sub + q * TPR], yv[sub + q * TPR], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if constexpr (TPR > 32) {
      if ((tid & 31) == 0) part[row][sub >> 5] = acc;
      __syncthreads();
      if (sub == 0) {
        double t = 0.0;
        for (int w = 0; w < TPR / 32; ++w) t += part[row][w];
        ybuf[(size_t)(s + 1) * kN + blockIdx.x * R + row] = t * 1e-3;
      }
    } else {
      if (sub == 0) ybuf[(size_t)(s + 1) * kN + blockIdx.x * R + row] = acc * 1e-3;
    }
    __syncthreads();
  }
  if (tid == 0) cyc[blockIdx.x] = clock64() - t0;
}

template <int R>
void run(int steps) {
  const int C = kN / R;
  double *ybuf, *A;
  long long* cyc;
  cudaMalloc(&ybuf, sizeof(double) * kN * (steps + 1));
  cudaMalloc(&A, sizeof(double) * (size_t)kN * kK);
  cudaMalloc(&cyc, sizeof(long long) * C);
  std::vector<double> h((size_t)kN * kK);
  for (size_t i = 0; i < h.size(); ++i) h[i] = 1e-3 * ((i * 2654435761u) % 1000) / 1000.0;
  cudaMemcpy(A, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const size_t smem = sizeof(double) * (R * kK + kK);
  cudaFuncSetAttribute(superchain<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemset(ybuf, 0xff, sizeof(double) * kN * (steps + 1));
    std::vector<double> y0(kN, 0.5);
    cudaMemcpy(ybuf, y0.data(), kN * 8, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    superchain<R><<<C, 512, smem>>>(ybuf, A, steps, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c0;
    cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
    printf("C=%3d CTAs (R=%2d rows): %s  %d steps  %.2f us total  %.3f us/step  (%lld cycles/step in-kernel)\n", C, R,
           cudaGetErrorString(cudaGetLastError()), steps, ms * 1e3, ms * 1e3 / steps, c0 / steps);
  }
}

int main() {
  run<4>(64);
  run<8>(64);
  run<16>(64);
  run<32>(64);
  return 0;
}
