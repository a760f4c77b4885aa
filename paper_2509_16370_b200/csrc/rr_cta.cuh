// rr_cta.cuh -- launch interface of the CTA-per-instance kernel for large stages (rr_cta.cu).
#pragma once
#include "rr_fused.cuh"

namespace rrk {
int64_t cta_workspace_bytes(int nx, int nu, int N, int64_t batch);
cudaError_t cta_launch(const FusedArgs& a, cudaStream_t s, bool* supported);
}  // namespace rrk
