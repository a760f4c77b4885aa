// rr_fused.cuh -- internal launch interface of the fused Riccati kernel (rr_fused.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rr.h"

namespace rrk {

struct FusedArgs {
  int nx, nu, N;
  int64_t batch;
  rr_problem p;
  rr_factor_buf f;
  rr_solution s;
  double* ws;
  int32_t* status;
  double* frec = nullptr;  // rr_factor on the DMMA kernel: factor records [batch][N+1][frec_doubles]
  float* frec32 = nullptr; // ... or FP32 records [batch][N+1][frec_floats] (RR_FLAG_FACTOR_FP32)
  int shared = 0;          // RR_FLAG_SHARED_DYN | RR_FLAG_SHARED_COST (batch-shared operands)
  // every stage-operand base pointer (A, B, Q, M, R, q, r, c) is 16-byte aligned: the TMA
  // (cp.async.bulk) kernels may run; otherwise the 12x4 shape falls back to the LDGSTS kernel
  // (8-byte copies where needed) and the CTA kernels are refused by the API (rr_api.cu)
  bool tma16 = true;
  // DMMA kernel (persistent warps): SM count and the phase-staggering modulus (set by the launcher)
  int nsm = 0, defer_mod = 1;
};

// Bytes of workspace for this shape (-1 if no kernel is compiled for it).
int64_t fused_workspace_bytes(int nx, int nu, int N, int64_t batch);
// Launch on stream s; *supported = false if no kernel covers (nx, nu).
cudaError_t fused_launch(const FusedArgs& a, cudaStream_t s, bool* supported);
// rr_factor on the DMMA stage kernel (factor-only mode); *supported = false outside its shapes.
cudaError_t factor_mma_launch(const FusedArgs& a, cudaStream_t s, bool* supported);

}  // namespace rrk
