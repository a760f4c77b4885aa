// rr_pit.cuh -- internal launch interface of the parallel-in-time solve (rr_pit.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rr.h"

namespace rrk {

struct PitArgs {
  int nx, nu, N;
  int64_t batch;
  rr_problem p;
  rr_solution s;
  double* ws;
  int32_t* status;
  int shared;  // RR_FLAG_SHARED_DYN | RR_FLAG_SHARED_COST
  int refine;  // FP64 iterative-refinement steps after the reduction solve
  // the reduction solves the system at δ_s = max(δ, delta_floor) (conditioning of the δ-scaled state
  // system ~ 1/δ_s); the refinement residuals use the caller's δ, so iterated refinement converges to
  // the solution at δ (δ = 0 included) -- contraction per step ≈ δ_s · ||(C P⁻¹ Cᵀ)⁻¹|| on the tests
  double delta_floor;
};

int64_t pit_ws_bytes(int nx, int nu, int N, int64_t batch);
cudaError_t pit_launch(const PitArgs& a, cudaStream_t s);

}  // namespace rrk
