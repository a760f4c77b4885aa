// DMMA (mma.sync.m8n8k4.f64) latency / issue probe on one warp: dependent chains of C accumulators
// (C = 1, 2, 4, 8), cycles per DMMA; and the same with the A/B fragments loaded from shared memory
// through the swizzled index of the C3 kernel (swz<64>) each step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dmma_probe.cu -o tools/dmma_probe
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int C>
__global__ void chain(double* out, long long* cyc, int R) {
  double c[C][2];
  for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = threadIdx.x;
  const double a = 1.0000001, b = 0.9999999;
  long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
#pragma unroll
    for (int i = 0; i < C; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
  for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
__device__ __forceinline__ int swz(int r, int c) { return c * 64 + (r ^ (((c ^ (c >> 2)) & 3) << 2)); }
// 16×16 tile, K = 64 from swizzled shared memory (the C3 kernel's warp tile), repeated R times
__global__ void tile(double* out, long long* cyc, int R) {
  __shared__ double A[64 * 32], B[64 * 32];
  for (int e = threadIdx.x; e < 64 * 32; e += blockDim.x) {
    A[e] = 1e-3 * (e % 7);
    B[e] = 1e-3 * (e % 5);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double c[2][2][2] = {};
  long long t0 = clock64();
  for (int r = 0; r < R; ++r) {
#pragma unroll 4
    for (int kt = 0; kt < 16; ++kt) {
      double av[2], bv[2];
#pragma unroll
      for (int a = 0; a < 2; ++a) av[a] = A[swz(8 * a + g, 4 * kt + t)];
#pragma unroll
      for (int b = 0; b < 2; ++b) bv[b] = B[(8 * b + g) * 64 + ((4 * kt + t) ^ ((((8 * b + g) ^ ((8 * b + g) >> 2)) & 3) << 2))];
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) dmma(c[a][b][0], c[a][b][1], av[a], bv[b]);
    }
  }
  long long t1 = clock64();
  double s = 0;
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b) s += c[a][b][0] + c[a][b][1];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 64);
  const int R = 4096;
  long long h;
  auto run = [&](auto kern, int threads, const char* name, double per) {
    kern<<<1, threads>>>(out, cyc, R);
    kern<<<1, threads>>>(out, cyc, R);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-48s %8.2f cycles per %s\n", name, (double)h / (R * per), per == 1 ? "iteration" : "DMMA");
  };
  run(chain<1>, 32, "1 warp, 1 dependent chain", 1);
  run(chain<2>, 32, "1 warp, 2 chains", 2);
  run(chain<4>, 32, "1 warp, 4 chains", 4);
  run(chain<8>, 32, "1 warp, 8 chains", 8);
  run(chain<8>, 128, "4 warps (1/SMSP), 8 chains each (per warp)", 8);
  run(chain<8>, 512, "16 warps, 8 chains each (per warp)", 8);
  run(tile, 32, "1 warp: 16x16 tile K=64 from swizzled smem", 64);
  run(tile, 512, "16 warps: 16x16 tile K=64 each (per warp)", 64);
  return 0;
}
