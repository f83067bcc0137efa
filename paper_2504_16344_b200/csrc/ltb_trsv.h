// ltb_trsv.h -- K^{-1} application through the dense lower Cholesky factor
// (replaces InferenceEngine::solve_k_inplace, bayes_engine.cpp:236-240:
// Eigen triangularView<Lower>().solveInPlace then its transpose), on one GPU
// or distributed over P GPUs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "ltb_nccl.h"

namespace ltb {

constexpr int kTB = 64;        // factor tile edge
constexpr int kMaxLook = 8;    // diagonal-chain lookahead depth bound (chain terms = chain CTAs)
// Chain depth for nb blocks: 8 terms (a cluster of 8 chain CTAs) where the
// sequential chain dominates (small n: the workers get 8 steps of slack), 4
// where panel streaming dominates (clusters of 8 leave only 120 of 148 SMs
// co-resident).  Every rank of a distributed factor picks the same depth.
inline int trsv_look_for(int nb) { return nb <= 256 ? 8 : 4; }
constexpr int kMaxRanks = 8;
// one GPU up to this many 64-blocks solves through the super-block chain
// (8 blocks per chain step); beyond, streaming the panel dominates and the
// head/tail chain kernel runs
constexpr int kSuperMaxNb = 512;

// Row-cyclic block distribution over P ranks: rank r holds the 64-row block
// rows I = r, r+P, r+2P, ... packed row after row (row I has I+1 tiles,
// local row li = (I-r)/P starts at tile li (r+1) + P li (li-1)/2; tiles are
// column-major 64x64).  P = 1 is the plain packed lower triangle.  The last
// block row / column is padded with the identity.
//
// Precomputed at set_factor time (every rank): dinv[I] = L_II^{-1} for ALL
// I; on rank 0 (the chain rank) the chain tiles
//   mf[I][k-1] = L_II^{-1} L_{I,I-k},  mb[I][k-1] = L_II^{-T} L_{I+k,I}^T.
//
// `recv` is the one allocation other ranks write into (CUDA IPC exported):
// [ yf | xb | ready (8 doubles) | cf | cb (P blocks) ], each vector nb*64.
struct TriFactor {
  int n = 0, nb = 0, P = 1, rank = 0;
  int look = 4;  // chain depth (trsv_look_for)
  double* tiles = nullptr;
  double* dinv = nullptr;
  double* mf = nullptr;
  double* mb = nullptr;
  double* recv = nullptr;
  double* peer_recv[kMaxRanks] = {};  // every rank's recv as addressable here
  bool peer_opened[kMaxRanks] = {};
  unsigned* gsync = nullptr;  // local grid barrier words
  int* status = nullptr;      // device error word (spin timeout / bad pivot)
  unsigned long long* trace = nullptr;  // diagnostic timestamps, 4 nb + 1 (optional)
  // P = 1, nb <= kSuperMaxNb: rows [L_SS^{-1} | -M_S] / [L_SS^{-T} | -M'_S]
  // of the super-block chain (ltb_trsv.cu trsv_super_kernel), ns blocks
  double* sfwd = nullptr;
  double* sbwd = nullptr;
  double* spart = nullptr;  // the workers' partial sums
  void* stasks = nullptr;   // their task list (int4 each)
  int nstasks = 0;
  int ns = 0;
  unsigned epoch = 0;
  size_t bytes = 0;
};

// n = N_d * N_t, P ranks, this rank
cudaError_t trsv_alloc(TriFactor& t, int n, int P = 1, int rank = 0);
void trsv_free(TriFactor& t);
// P == 1: pack from a device column-major matrix (only the lower triangle
// is read), then trsv_prepare_packed
cudaError_t trsv_pack_colmajor(TriFactor& t, const double* L, size_t ld, cudaStream_t st);
cudaError_t trsv_prepare_packed(TriFactor& t, cudaStream_t st);
// any P: pack this rank's rows of the synthetic factor (ltb_gen.cuh
// gen_factor_entry) and build dinv / chain tiles from regenerated tiles
cudaError_t trsv_setup_generated(TriFactor& t, uint64_t seed, cudaStream_t st);
// A real distributed factor in t.tiles (ltb_formk.h cholesky_dist): dinv for
// every block from the all-gathered diagonal tiles, chain tiles computed by the
// owner of each L tile and gathered on rank 0 (collective over comm).
cudaError_t trsv_prepare_dist(TriFactor& t, const Nccl* api, ncclComm_t comm, cudaStream_t st, const char** err);
// P > 1: exchange `recv` (CUDA IPC); handles[p] for every rank
cudaError_t trsv_ipc_handle(const TriFactor& t, cudaIpcMemHandle_t* out);
cudaError_t trsv_connect(TriFactor& t, const cudaIpcMemHandle_t* handles);
// x = L^{-T} L^{-1} b for b of length nb*64 (zero padded, the same on every
// rank); the result is left in trsv_result(t) on EVERY rank.  One
// cooperative launch per rank; ranks must launch concurrently.
cudaError_t trsv_solve(TriFactor& t, const double* b, cudaStream_t st);
double* trsv_result(TriFactor& t);
// Process-wide lock of device `dev` for the persistent K^{-1} launch: the
// kernel fills the GPU and needs all of its CTAs resident, so two of them
// must never run at once.  Callers hold it from the launch until they have
// synchronized the launch stream.
std::mutex& trsv_device_mutex(int dev);
// All P ranks emulated by ONE cooperative launch on the current GPU (test /
// validation of the distributed algorithm without P GPUs).
cudaError_t trsv_solve_emulated(TriFactor* const* ts, const double* const* bs, int P,
                                cudaStream_t st);

}  // namespace ltb
