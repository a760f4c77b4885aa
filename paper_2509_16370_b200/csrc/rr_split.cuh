// rr_split.cuh -- internal launch interface of the rr_factor / rr_solve kernels (rr_split.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rr.h"

namespace rrk {

struct SplitArgs {
  int nx, nu, N;
  int64_t batch;
  rr_problem p;
  rr_factor_buf f;   // optional user copies (rr_factor: V, K; rr_solve: v, k)
  rr_solution s;     // rr_solve outputs
  double* fr;        // rr_factor: factor records [batch][N+1][frec_doubles]
  const double* frc; // rr_solve: the same records, read only
  double* ws;        // rr_solve scratch: [batch][N][n+m] (v_i | k_i)
  int32_t* status;
  int accumulate;    // rr_solve: RR_FLAG_ACCUMULATE (sol += solution)
  int shared;        // RR_FLAG_SHARED_DYN | RR_FLAG_SHARED_COST
  bool tma16;        // rr_factor: A, B, Q, M, R 16-byte aligned (the 12x4 DMMA/TMA factor kernel may run)
  bool f32;          // RR_FLAG_FACTOR_FP32: FP32 factor records (12x4 only)
};

struct ResArgs {
  int nx, nu, N;
  int64_t batch;
  rr_problem p;
  rr_solution s;     // candidate (read)
  rr_residual_buf r; // residual blocks (any member may be null)
  double* norms;     // [batch][2] or null
  int shared;        // RR_FLAG_SHARED_DYN | RR_FLAG_SHARED_COST
};

// doubles per factor record: V (packed n) | S⁻¹ (packed n) | K (m×n) | G⁻¹ (packed m), even
__host__ __device__ inline int frec_doubles(int n, int m) {
  return (n * (n + 1) + n * m + m * (m + 1) / 2 + 1) & ~1;
}

// floats per FP32 factor record (RR_FLAG_FACTOR_FP32): the same layout, rounded to a 16-byte multiple
__host__ __device__ inline int frec_floats(int n, int m) { return (frec_doubles(n, m) + 3) & ~3; }

bool split_supported(int nx, int nu);
cudaError_t factor_launch(const SplitArgs& a, cudaStream_t s, bool* supported);
cudaError_t solve_launch(const SplitArgs& a, cudaStream_t s, bool* supported);
cudaError_t residual_launch(const ResArgs& a, cudaStream_t s, bool* supported);

}  // namespace rrk
