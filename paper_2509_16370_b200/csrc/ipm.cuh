// ipm.cuh -- internal launch interface of the fused ipm_step kernel (ipm.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rr.h"

namespace rrk {

struct IpmArgs {
  ipm_dims d;
  ipm_stage_data d_;
  ipm_iterate it;
  ipm_params prm;
  ipm_result r;
  double* ws;
  int32_t* status;
  const int32_t* list = nullptr;   // ipm_solve: active instance ids (nullptr: all instances)
  const int32_t* count = nullptr;  // device count of `list`
  int direction_only = 0;          // ipm_direction: rows a1-a7 only (no line search, no update)
  int aligned16 = 0;               // set by ipm_launch: 16-byte aligned operand bases (C4 copy plan)
};

int64_t ipm_ws_bytes(const ipm_dims& d);
cudaError_t ipm_launch(const IpmArgs& a, cudaStream_t s, bool* supported);
bool ipm_supported(const ipm_dims& d);
// the C4 shape on one thread per instance (ipm_c4t.cu)
bool ipm_c4t_applies(const IpmArgs& a);
cudaError_t ipm_c4t_launch(const IpmArgs& a, cudaStream_t s);
// caller-evaluated line search (ipm_user.cu)
cudaError_t ipm_merit_launch(const ipm_dims& d, const ipm_stage_data& data, const ipm_iterate& it, const ipm_result& r,
                             const double* alpha, const ipm_trial_values& tv, double* merit, cudaStream_t s);
cudaError_t ipm_update_launch(const ipm_dims& d, const ipm_iterate& it, const ipm_result& r, const double* alpha_p,
                              const double* alpha_d, cudaStream_t s);

}  // namespace rrk
