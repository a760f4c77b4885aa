// ipm_solve.cuh -- internal launch interface of the batched IPM solve (ipm_solve.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "rr.h"

namespace rrk {
int64_t ipm_solve_ws_bytes(const ipm_dims& d);
cudaError_t ipm_solve_launch(const ipm_dims& d, const ipm_stage_data& data, const ipm_iterate& it,
                             const ipm_solve_settings& S, const ipm_solve_report& rep, void* workspace,
                             cudaStream_t s, bool* supported);
}  // namespace rrk
