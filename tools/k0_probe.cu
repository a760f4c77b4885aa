// K0 probe (standalone): FP64 DFMA and DMMA (mma.sync m8n8k4 f64) throughput on this GPU.
// Used to pick the kernel design; `bench.py --workload c3` builds and runs it to measure the FP64
// DMMA roofline peak in the same run.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = threadIdx.x * 1e-3 + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = fma(acc[j], a, b);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-6, b = 0.5;
  double c[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) { c[j][0] = 0; c[j][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[0] = s;
}

// Broadcast LDS.128 throughput: every lane of a half-warp reads the same 16 B.
__global__ void lds_kernel(double* out, int iters) {
  __shared__ double2 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_double2(i, i + 1);
  __syncthreads();
  double s0 = 0, s1 = 0;
  int base = (threadIdx.x >> 4) & 1;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      double2 v = buf[(j * 2 + base + it) & 1023];
      s0 += v.x; s1 += v.y;
    }
  }
  if (s0 + s1 == 12345.678) out[0] = s0;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* d; cudaMalloc(&d, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int rep = 0; rep < 3; ++rep) {
    int iters = 1 << 14, threads = 256, blocks = sms * 8;
    dfma_kernel<<<blocks, threads>>>(d, 16, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * (double)iters * threads * blocks;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);

    dmma_kernel<<<blocks, threads>>>(d, 16);
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 256 * 4 * (double)iters * (threads / 32) * blocks;
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);

    lds_kernel<<<blocks, threads>>>(d, 16);
    cudaEventRecord(e0);
    lds_kernel<<<blocks, threads>>>(d, iters / 4);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double lds = 16.0 * (iters / 4) * (threads / 32) * blocks;
    printf("LDS.128 (2 addr/warp): %.3f Tinstr/s = %.2f per SM per ns (%.3f ms)\n", lds / ms / 1e9,
           lds / ms / 1e6 / sms, ms);
  }
  cudaError_t err = cudaGetLastError();
  printf("err: %s\n", cudaGetErrorString(err));
  return 0;
}
