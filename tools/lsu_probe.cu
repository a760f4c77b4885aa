// Throughput probe of the shared-memory / shuffle paths the 12x4 kernel is bound by (B200).
// Per variant: 16 warps per SM x 148 SMs, each warp issues R loads of one pattern; prints SM cycles
// per warp-instruction (1 SM, clock64) -- i.e. the LSU cost of one instruction of that pattern.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/lsu_probe.cu -o /tmp/lsu_probe
#include <cstdio>
#include <cstdint>
#define R 2048
template <int V>
__global__ void probe(double* out, long long* cyc) {
  __shared__ __align__(16) double sm[4096];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i * 0.5;
  __syncthreads();
  double acc0 = 0, acc1 = 0;
  int off = 0;
  long long t0 = clock64();
#pragma unroll 8
  for (int r = 0; r < R; ++r) {
    off = (r * 16) & 1023;
    if (V == 0) {  // LDS.128, all 32 lanes same address (full broadcast)
      double2 v = *reinterpret_cast<const double2*>(sm + off);
      acc0 += v.x; acc1 += v.y;
    } else if (V == 1) {  // LDS.128, two addresses (half-warps), 16 doubles apart
      double2 v = *reinterpret_cast<const double2*>(sm + off + 16 * (lane >> 4) + 8 * w);
      acc0 += v.x; acc1 += v.y;
    } else if (V == 2) {  // LDS.64 full broadcast
      acc0 += sm[off];
    } else if (V == 3) {  // LDS.64 two addresses (half-warps)
      acc0 += sm[off + 16 * (lane >> 4) + 8 * w];
    } else if (V == 4) {  // LDS.64 32 distinct consecutive (conflict-free)
      acc0 += sm[off + lane];
    } else if (V == 5) {  // LDS.128 32 distinct consecutive
      double2 v = *reinterpret_cast<const double2*>(sm + off + 2 * lane);
      acc0 += v.x; acc1 += v.y;
    } else if (V == 6) {  // SHFL of a double (2 x SHFL.IDX)
      acc0 += __shfl_sync(0xffffffffu, acc1 + r, (lane + r) & 31);
    } else if (V == 7) {  // LDS.128, four addresses (quarter-warps... lanes>>3)
      double2 v = *reinterpret_cast<const double2*>(sm + off + 16 * (lane >> 3) + 8 * w);
      acc0 += v.x; acc1 += v.y;
    } else if (V == 8) {  // STS.64 32 distinct consecutive
      sm[2048 + ((off + lane + 32 * w) & 2047)] = acc0 + r;
    } else if (V == 9) {  // STS.128 32 distinct consecutive
      *reinterpret_cast<double2*>(sm + 2048 + ((off + 2 * lane + 64 * w) & 2047)) = make_double2(acc0 + r, acc1);
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  if (acc0 + acc1 == 1234.5) out[0] = acc0;
}
template <int V>
void run(const char* name, double* out, long long* cyc) {
  probe<V><<<148, 512>>>(out, cyc);
  cudaDeviceSynchronize();
  probe<V><<<148, 512>>>(out, cyc);
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double m = 0;
  for (int i = 0; i < 148; ++i) m += h[i];
  m /= 148;
  printf("%-40s %.3f SM-cycles per warp-instruction (16 warps/SM)\n", name, m / (R * 16.0));
}
int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 148 * 8);
  run<0>("LDS.128 full broadcast", out, cyc);
  run<1>("LDS.128 2 addresses (half-warps)", out, cyc);
  run<7>("LDS.128 4 addresses (quarter-warps)", out, cyc);
  run<2>("LDS.64 full broadcast", out, cyc);
  run<3>("LDS.64 2 addresses (half-warps)", out, cyc);
  run<4>("LDS.64 32 distinct", out, cyc);
  run<5>("LDS.128 32 distinct", out, cyc);
  run<6>("SHFL double (2 x SHFL.IDX)", out, cyc);
  run<8>("STS.64 32 distinct", out, cyc);
  run<9>("STS.128 32 distinct", out, cyc);
  return 0;
}
