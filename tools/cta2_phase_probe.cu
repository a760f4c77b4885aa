// Phase timeline of the C3 K4b kernel (two CTAs per SM; tools/cta_phase_probe.cu is the K4 twin): builds rr_cta.cu with RR_CTA_PROFILE=<stage> so CTA 0 records
// clock64() at the phase boundaries of that stage (and of the forward sweep), runs one full wave of
// C3-shaped instances (n_x = 64, n_u = 32, N = 50) on synthetic well-conditioned data, prints cycles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DRR_CTA_PROFILE=25 -I include
//        -I paper_2509_16370_b200/csrc tools/cta_phase_probe.cu -o tools/cta_phase_probe
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "rr_cta.cu"

int main() {
  constexpr int NX = 64, NU = 32, N = 50;
  const int64_t B = 296;
  using L = rrk::CtaLayout<NX, NU>;
  auto fill = [](std::vector<double>& v, double scale, unsigned seed) {
    srand(seed);
    for (auto& x : v) x = scale * (rand() / (double)RAND_MAX - 0.5);
  };
  std::vector<double> A(B * N * NX * NX), Bm(B * N * NX * NU), Q(B * N * L::SN), M(B * N * NX * NU),
      R(B * N * L::SMU), q(B * N * NX), r(B * N * NU), c(B * N * NX), QN(B * L::SN), qN(B * NX), c0(B * NX),
      delta(B, 1e-4);
  fill(A, 0.1, 1); fill(Bm, 0.2, 2); fill(M, 0.01, 3); fill(q, 1, 4); fill(r, 1, 5); fill(c, 1, 6);
  fill(qN, 1, 7); fill(c0, 1, 8);
  for (int64_t s = 0; s < B * N; ++s) {
    for (int i = 0; i < NX; ++i) A[s * NX * NX + i + i * NX] += 0.95;
    for (int cc = 0; cc < NX; ++cc)
      for (int rr = cc; rr < NX; ++rr) Q[s * L::SN + rrk::pidx(NX, rr, cc)] = rr == cc ? 1.0 : 0.0;
    for (int cc = 0; cc < NU; ++cc)
      for (int rr = cc; rr < NU; ++rr) R[s * L::SMU + rrk::pidx(NU, rr, cc)] = rr == cc ? 1.0 : 0.0;
  }
  for (int64_t b = 0; b < B; ++b)
    for (int cc = 0; cc < NX; ++cc)
      for (int rr = cc; rr < NX; ++rr) QN[b * L::SN + rrk::pidx(NX, rr, cc)] = rr == cc ? 1.0 : 0.0;
  auto up = [](const std::vector<double>& h) {
    double* d;
    cudaMalloc(&d, h.size() * sizeof(double));
    cudaMemcpy(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice);
    return d;
  };
  rrk::FusedArgs a{};
  a.nx = NX; a.nu = NU; a.N = N; a.batch = B;
  a.p.A = up(A); a.p.B = up(Bm); a.p.Q = up(Q); a.p.M = up(M); a.p.R = up(R); a.p.q = up(q); a.p.r = up(r);
  a.p.c = up(c); a.p.QN = up(QN); a.p.qN = up(qN); a.p.c0 = up(c0); a.p.delta = up(delta);
  cudaMalloc(&a.s.x, B * (N + 1) * NX * sizeof(double));
  cudaMalloc(&a.s.u, B * N * NU * sizeof(double));
  cudaMalloc(&a.s.y, B * (N + 1) * NX * sizeof(double));
  cudaMalloc(&a.ws, B * N * L::REC * sizeof(double));
  cudaMalloc(&a.status, B * sizeof(int32_t));
  using Cfg = rrk::Cta2Cfg<NX, NU>;
  for (int rep = 0; rep < 3; ++rep) Cfg::launch(a, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  Cfg::launch(a, 0);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long t[32];
  cudaMemcpyFromSymbol(t, rrk::g_cta_prof, sizeof t);
  std::vector<int32_t> st(B);
  cudaMemcpy(st.data(), a.status, B * 4, cudaMemcpyDeviceToHost);
  int nbad = 0;
  for (auto v : st) nbad += v != 0;
  printf("err=%s  one wave (296 instances, N=%d): %.3f ms = %.1f us/stage  status!=0: %d\n", cudaGetErrorString(err),
         N, ms, ms * 1e3 / N, nbad);
  const char* names[] = {"S=I+dV, e, Ve", "S sweep", "W = S^-1 V, g, rec S^-1", "T = W F (T_A from L2)", "G, H, b",
                         "G sweep | Uxx", "K~, k~", "V_i, v_i"};
  for (int k = 0; k < 8; ++k) printf("  %-28s %7lld cyc\n", names[k], t[k + 1] - t[k]);
  printf("  stage total (slot 0..8)      %7lld cyc\n", t[8] - t[0]);
  for (int p = 0; p < 4; ++p)
    printf("    S block %d: diag %6lld  Y %6lld  trailing %6lld\n", p, t[13 + 3 * p] - t[12 + 3 * p],
           t[14 + 3 * p] - t[13 + 3 * p], (p < 3 ? t[15 + 3 * p] : t[2]) - t[14 + 3 * p]);
  printf("  x0 solve                     %7lld cyc\n", t[10] - t[9]);
  printf("  forward sweep (%d stages)    %7lld cyc = %.0f cyc/stage\n", N, t[11] - t[10], (t[11] - t[10]) / (double)N);
  return 0;
}
