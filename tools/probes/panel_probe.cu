// Phase timing of the tile-Cholesky panel kernel (CTA 0, clock64 stamps):
// load / per 16-column block (diagonal factor, row solve, DMMA update) /
// store.  Builds ltb_formk.cu into this TU with the stamps compiled in.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2504_16344_b200/csrc tools/probes/panel_probe.cu -o tools/probes/panel_probe
#define LTB_PANEL_STAMPS 1
#include "ltb_formk.cu"

#include <cstdio>

int main() {
  using namespace ltb;
  const int nb = 8;
  const size_t ntile = (size_t)nb * (nb + 1) / 2 * kTile;
  std::vector<double> h(ntile, 0.0);
  // K = diagonally dominant SPD: 2 n on the diagonal, 1 / (1 + |i - j|) off it
  const int n = nb * kT;
  for (int I = 0; I < nb; ++I)
    for (int J = 0; J <= I; ++J)
      for (int c = 0; c < kT; ++c)
        for (int r = 0; r < kT; ++r) {
          const int i = I * kT + r, j = J * kT + c;
          h[tile_at(I, J) + c * kT + r] = i == j ? 2.0 * n : 1.0 / (1 + abs(i - j));
        }
  double* d;
  int* st;
  cudaMalloc(&d, ntile * sizeof(double));
  cudaMalloc(&st, sizeof(int));
  cudaMemset(st, 0, sizeof(int));
  cudaFuncSetAttribute(chol_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPanelSmem);
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d, h.data(), ntile * sizeof(double), cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chol_panel_kernel<<<nb - 1, kPanelThreads, kPanelSmem>>>(d, nb, 0, st);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long s[32];
    cudaMemcpyFromSymbol(s, g_pstamp, sizeof(s));
    printf("rep %d: %s  kernel %.2f us; cycles: load %lld", rep, cudaGetErrorString(cudaGetLastError()),
           ms * 1e3, s[1] - s[0]);
    for (int b = 0; b < 4; ++b)
      printf(" | b%d diag %lld solve %lld upd %lld", b, s[2 + 3 * b] - (b ? s[1 + 3 * b] : s[1]),
             s[3 + 3 * b] - s[2 + 3 * b], s[4 + 3 * b] - s[3 + 3 * b]);
    printf(" | store %lld total %lld\n", s[15] - s[14], s[15] - s[0]);
  }
  return 0;
}
