// Latency probe for the 16×16 warp-register symmetric sweep (the serial chain of the C3 block sweep).
// One warp per block, clock64 around R repetitions; prints cycles per 16-pivot sweep per variant and
// the max deviation from variant 0.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I
// paper_2509_16370_b200/csrc tools/sweep_probe.cu -o /tmp/sweep_probe
#include <cstdio>
#include <cmath>
#include "rr_common.cuh"
using namespace rrk;

// V0: lane = (column c = l & 15, rows 8h..8h+7)
__device__ __forceinline__ void sweep_v0(double (&a)[8], int lane) {
  const int c = lane & 15, h = lane >> 4;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const double d = __shfl_sync(RR_FULL_MASK, a[k & 7], k + 16 * (k >> 3));
    const double rowk = __shfl_sync(RR_FULL_MASK, a[k & 7], c + 16 * (k >> 3));
    double colk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) colk[i] = __shfl_sync(RR_FULL_MASK, a[i], k + 16 * h);
    const double id = rcp_nr(d);
    const double rs = rowk * id;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 8 * h + i;
      const double upd = fma(-colk[i], rs, a[i]);
      a[i] = (r == k) ? ((c == k) ? -id : rs) : ((c == k) ? colk[i] * id : upd);
    }
  }
}

// V1: lane = (row group rg = l >> 3: rows 4rg..4rg+3, column pair cp = l & 7: cols 2cp, 2cp+1);
// a[i][j] = A[4rg+i][2cp+j].  7 shuffles per pivot instead of 10.
__device__ __forceinline__ void sweep_v1(double (&a)[4][2], int lane) {
  const int rg = lane >> 3, cp = lane & 7;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int kr = k >> 2, ki = k & 3, kc = k >> 1, kj = k & 1;
    const double d = __shfl_sync(RR_FULL_MASK, a[ki][kj], kr * 8 + kc);
    double colk[4], rowk[2];
#pragma unroll
    for (int i = 0; i < 4; ++i) colk[i] = __shfl_sync(RR_FULL_MASK, a[i][kj], rg * 8 + kc);  // A[4rg+i][k]
#pragma unroll
    for (int j = 0; j < 2; ++j) rowk[j] = __shfl_sync(RR_FULL_MASK, a[ki][j], kr * 8 + cp);  // A[k][2cp+j]
    const double id = rcp_nr(d);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int c = 2 * cp + j;
      const double rs = rowk[j] * id;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = 4 * rg + i;
        const double upd = fma(-colk[i], rs, a[i][j]);
        a[i][j] = (r == k) ? ((c == k) ? -id : rs) : ((c == k) ? colk[i] * id : upd);
      }
    }
  }
}

// V2: V0 layout, pivots in 2×2 blocks: Z = D⁻¹ (D = [[p q]; [q s]]), one reciprocal per pair.
__device__ __forceinline__ void sweep_v2(double (&a)[8], int lane) {
  const int c = lane & 15, h = lane >> 4;
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const int o = 16 * (k >> 3);
    const double p = __shfl_sync(RR_FULL_MASK, a[k & 7], k + o);
    const double q = __shfl_sync(RR_FULL_MASK, a[k & 7], k + 1 + o);
    const double sd = __shfl_sync(RR_FULL_MASK, a[(k + 1) & 7], k + 1 + o);
    const double r0 = __shfl_sync(RR_FULL_MASK, a[k & 7], c + o);        // A[k][c]
    const double r1 = __shfl_sync(RR_FULL_MASK, a[(k + 1) & 7], c + o);  // A[k+1][c]
    double c0[8], c1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      c0[i] = __shfl_sync(RR_FULL_MASK, a[i], k + 16 * h);
      c1[i] = __shfl_sync(RR_FULL_MASK, a[i], k + 1 + 16 * h);
    }
    const double idet = rcp_nr(fma(p, sd, -q * q));
    const double z00 = sd * idet, z01 = -q * idet, z11 = p * idet;
    const double zr0 = fma(z00, r0, z01 * r1), zr1 = fma(z01, r0, z11 * r1);  // (Z [A_k; A_k+1])[:, c]
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 8 * h + i;
      const double upd = fma(-c1[i], zr1, fma(-c0[i], zr0, a[i]));
      const double ck = fma(c0[i], z00, c1[i] * z01), ck1 = fma(c0[i], z01, c1[i] * z11);
      double v = upd;
      if (c == k) v = ck;
      if (c == k + 1) v = ck1;
      if (r == k) v = (c == k) ? -z00 : ((c == k + 1) ? -z01 : zr0);
      if (r == k + 1) v = (c == k) ? -z01 : ((c == k + 1) ? -z11 : zr1);
      a[i] = v;
    }
  }
}

__global__ void probe(double* out, long long* cyc, int R) {
  const int lane = threadIdx.x;
  // SPD test matrix: A = I*4 + small symmetric (r, c) pattern
  auto Af = [](int r, int c) { return (r == c ? 4.0 : 0.0) + 0.1 / (1.0 + r + c); };
  double res[3][256 / 32];
  long long t[3];
  {
    double a[8];
    const int c = lane & 15, h = lane >> 4;
    long long t0 = clock64();
    for (int rep = 0; rep < R; ++rep) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = Af(8 * h + i, c) + rep * 1e-12;
      sweep_v0(a, lane);
      __syncwarp();
    }
    t[0] = clock64() - t0;
    for (int i = 0; i < 8; ++i) res[0][i] = a[i];
  }
  {
    double a[4][2];
    const int rg = lane >> 3, cp = lane & 7;
    long long t0 = clock64();
    for (int rep = 0; rep < R; ++rep) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) a[i][j] = Af(4 * rg + i, 2 * cp + j) + rep * 1e-12;
      sweep_v1(a, lane);
      __syncwarp();
    }
    t[1] = clock64() - t0;
    // remap to V0 ownership via shuffles: V0 lane (c, h) element i = A[8h+i][c]
    const int c = lane & 15, h = lane >> 4;
    for (int i = 0; i < 8; ++i) {
      const int r = 8 * h + i;
      double v = 0;
      for (int ii = 0; ii < 4; ++ii)
        for (int jj = 0; jj < 2; ++jj) {
          const double x = __shfl_sync(RR_FULL_MASK, a[ii][jj], (r >> 2) * 8 + (c >> 1));
          if (ii == (r & 3) && jj == (c & 1)) v = x;
        }
      res[1][i] = v;
    }
  }
  {
    double a[8];
    const int c = lane & 15, h = lane >> 4;
    long long t0 = clock64();
    for (int rep = 0; rep < R; ++rep) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = Af(8 * h + i, c) + rep * 1e-12;
      sweep_v2(a, lane);
      __syncwarp();
    }
    t[2] = clock64() - t0;
    for (int i = 0; i < 8; ++i) res[2][i] = a[i];
  }
  double dev1 = 0, dev2 = 0;
  for (int i = 0; i < 8; ++i) {
    dev1 = fmax(dev1, fabs(res[1][i] - res[0][i]));
    dev2 = fmax(dev2, fabs(res[2][i] - res[0][i]));
  }
  for (int off = 16; off > 0; off >>= 1) {
    dev1 = fmax(dev1, __shfl_xor_sync(RR_FULL_MASK, dev1, off));
    dev2 = fmax(dev2, __shfl_xor_sync(RR_FULL_MASK, dev2, off));
  }
  if (lane == 0) {
    for (int v = 0; v < 3; ++v) cyc[v] = t[v];
    out[0] = dev1;
    out[1] = dev2;
    out[2] = res[0][0];
  }
}

int main() {
  double* d_out;
  long long* d_cyc;
  cudaMalloc(&d_out, 3 * sizeof(double));
  cudaMalloc(&d_cyc, 3 * sizeof(long long));
  const int R = 2000;
  probe<<<1, 32>>>(d_out, d_cyc, R);
  double out[3];
  long long cyc[3];
  cudaMemcpy(out, d_out, sizeof out, cudaMemcpyDeviceToHost);
  cudaMemcpy(cyc, d_cyc, sizeof cyc, cudaMemcpyDeviceToHost);
  printf("cycles per 16-pivot sweep: v0 (8x1, 10 shfl) %.0f  v1 (4x2, 7 shfl) %.0f  v2 (2x2 pivots) %.0f\n",
         (double)cyc[0] / R, (double)cyc[1] / R, (double)cyc[2] / R);
  printf("max |v1 - v0| = %.3e   max |v2 - v0| = %.3e   (A00 after sweep %.6f)\n", out[0], out[1], out[2]);
  return 0;
}
