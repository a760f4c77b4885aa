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
};

int64_t ipm_ws_bytes(const ipm_dims& d);
cudaError_t ipm_launch(const IpmArgs& a, cudaStream_t s, bool* supported);
bool ipm_supported(const ipm_dims& d);

}  // namespace rrk
