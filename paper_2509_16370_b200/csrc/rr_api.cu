// rr_api.cu -- the C-ABI entry points declared in include/rr.h (host side: validation + launch).
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "rr.h"
#include "ipm.cuh"
#include "ipm_solve.cuh"
#include "rr_fused.cuh"
#include "rr_split.cuh"
#include "rr_pit.cuh"

namespace {
thread_local char g_err[512] = "";

rr_err set_err(rr_err code, const char* fmt, const char* what = "") {
  snprintf(g_err, sizeof(g_err), fmt, what);
  return code;
}

// operand-layout flags (batch-shared and stage-invariant A, B / Q, M, R; include/rr.h)
constexpr int SHARED_FLAGS =
    RR_FLAG_SHARED_DYN | RR_FLAG_SHARED_COST | RR_FLAG_STAGE_INVARIANT_DYN | RR_FLAG_STAGE_INVARIANT_COST;

// TMA bulk copies (cp.async.bulk) need 16-byte-aligned global addresses; the per-stage block
// offsets of every compiled TMA shape are multiples of 16 bytes, so the base pointers decide.
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool stage_ops_aligned16(const rr_problem* p) {
  const double* ops[] = {p->A, p->B, p->Q, p->M, p->R, p->q, p->r, p->c};
  for (const double* o : ops)
    if (!aligned16(o)) return false;
  return true;
}
bool large_shape(const rr_dims* d) { return d->nx > 16 || d->nu > 16; }  // CTA-per-instance kernels

bool dims_ok(const rr_dims* d, int allowed_flags = SHARED_FLAGS) {
  return d != nullptr && d->nx >= 1 && d->nu >= 1 && d->N >= 0 && d->batch >= 0 && (d->flags & ~allowed_flags) == 0;
}
}  // namespace

extern "C" {

const char* rr_last_error(void) { return g_err; }

const char* rr_version(void) { return "rr_b200 0.1 sm_100a"; }

int64_t rr_workspace_bytes(const rr_dims* dims) {
  if (!dims_ok(dims)) return -1;
  if ((dims->flags & SHARED_FLAGS) && (dims->nx > 16 || dims->nu > 16)) return -1;  // CTA kernels: per instance
  return rrk::fused_workspace_bytes(dims->nx, dims->nu, dims->N, dims->batch);
}

rr_err rr_factor_solve(const rr_dims* dims, const rr_problem* prob, const rr_factor_buf* fac,
                       const rr_solution* sol, void* workspace, int64_t workspace_bytes,
                       int32_t* status, void* stream) {
  if (!dims_ok(dims)) return set_err(RR_E_INVALID, "rr_factor_solve: invalid dims%s");
  if (prob == nullptr || sol == nullptr)
    return set_err(RR_E_INVALID, "rr_factor_solve: null %s", "prob/sol");
  if (dims->batch == 0) return RR_OK;  // nothing to do; status may be null for an empty batch
  if (status == nullptr) return set_err(RR_E_INVALID, "rr_factor_solve: null %s", "status");
  const double* req[] = {prob->QN, prob->qN, prob->c0, prob->delta};
  for (const double* p : req)
    if (p == nullptr) return set_err(RR_E_INVALID, "rr_factor_solve: null %s", "terminal/initial operand");
  if (dims->N > 0) {
    const double* req2[] = {prob->A, prob->B, prob->Q, prob->M, prob->R, prob->q, prob->r, prob->c};
    for (const double* p : req2)
      if (p == nullptr) return set_err(RR_E_INVALID, "rr_factor_solve: null %s", "stage operand");
  }
  if (sol->x == nullptr || sol->y == nullptr || (dims->N > 0 && sol->u == nullptr))
    return set_err(RR_E_INVALID, "rr_factor_solve: null %s", "solution pointer");
  const int64_t need = rr_workspace_bytes(dims);
  if (need < 0)
    return set_err(RR_E_UNSUPPORTED, "rr_factor_solve: no kernel compiled for this (nx, nu)%s");
  if (dims->N > 0 && (workspace == nullptr || workspace_bytes < need))
    return set_err(RR_E_INVALID, "rr_factor_solve: workspace missing or smaller than %s",
                   "rr_workspace_bytes()");
  if (!aligned16(workspace))
    return set_err(RR_E_INVALID, "rr_factor_solve: workspace not %s", "16-byte aligned");
  const bool tma16 = stage_ops_aligned16(prob);
  if (!tma16 && large_shape(dims) && dims->N > 0)
    return set_err(RR_E_INVALID, "rr_factor_solve: n or m > 16 needs %s",
                   "16-byte-aligned stage operands (TMA bulk copies of A, B)");
  rrk::FusedArgs a;
  a.nx = dims->nx;
  a.nu = dims->nu;
  a.N = dims->N;
  a.batch = dims->batch;
  a.p = *prob;
  rr_factor_buf none = {nullptr, nullptr, nullptr, nullptr};
  a.f = fac ? *fac : none;
  a.s = *sol;
  a.ws = static_cast<double*>(workspace);
  a.status = status;
  a.shared = dims->flags & SHARED_FLAGS;
  a.tma16 = tma16;
  bool supported = false;
  cudaError_t e = rrk::fused_launch(a, static_cast<cudaStream_t>(stream), &supported);
  if (!supported) return set_err(RR_E_UNSUPPORTED, "rr_factor_solve: unsupported shape%s");
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor_solve: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

rr_err rr_factor_solve_host(const rr_dims* dims, const rr_problem* ph, const rr_solution* sh,
                            int32_t* status_host, const rr_problem* pd, const rr_solution* sd,
                            int32_t* status_dev, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!dims_ok(dims)) return set_err(RR_E_INVALID, "rr_factor_solve_host: invalid dims%s");
  if (!ph || !sh || !pd || !sd || !status_host || !status_dev)
    return set_err(RR_E_INVALID, "rr_factor_solve_host: null %s", "argument");
  if (dims->batch == 0) return RR_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t b = dims->batch, N = dims->N, n = dims->nx, m = dims->nu;
  const int64_t sn = n * (n + 1) / 2, sm = m * (m + 1) / 2;
  const int64_t bD = (dims->flags & RR_FLAG_SHARED_DYN) ? 1 : b, bP = (dims->flags & RR_FLAG_SHARED_COST) ? 1 : b;
  const int64_t nD = (dims->flags & RR_FLAG_STAGE_INVARIANT_DYN) ? 1 : N;   // stage blocks of A, B
  const int64_t nP = (dims->flags & RR_FLAG_STAGE_INVARIANT_COST) ? 1 : N;  // stage blocks of Q, M, R
  struct Op { const double* h; const double* d; int64_t cnt; } ops[] = {
      {ph->A, pd->A, bD * nD * n * n}, {ph->B, pd->B, bD * nD * n * m}, {ph->Q, pd->Q, bP * nP * sn},
      {ph->M, pd->M, bP * nP * n * m}, {ph->R, pd->R, bP * nP * sm},    {ph->q, pd->q, b * N * n},
      {ph->r, pd->r, b * N * m},      {ph->c, pd->c, b * N * n},      {ph->QN, pd->QN, bP * sn},
      {ph->qN, pd->qN, b * n},       {ph->c0, pd->c0, b * n},       {ph->delta, pd->delta, b}};
  for (const Op& o : ops) {
    if (o.cnt == 0) continue;
    if (!o.h || !o.d) return set_err(RR_E_INVALID, "rr_factor_solve_host: null %s", "operand");
    cudaError_t e = cudaMemcpyAsync(const_cast<double*>(o.d), o.h, sizeof(double) * o.cnt,
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor_solve_host: H2D %s", cudaGetErrorString(e));
  }
  rr_err rc = rr_factor_solve(dims, pd, nullptr, sd, workspace, workspace_bytes, status_dev, stream);
  if (rc != RR_OK) return rc;
  struct Out { double* h; const double* d; int64_t cnt; } outs[] = {
      {sh->x, sd->x, b * (N + 1) * n}, {sh->u, sd->u, b * N * m}, {sh->y, sd->y, b * (N + 1) * n}};
  for (const Out& o : outs) {
    if (o.cnt == 0 || o.h == nullptr) continue;
    cudaError_t e = cudaMemcpyAsync(o.h, o.d, sizeof(double) * o.cnt, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor_solve_host: D2H %s", cudaGetErrorString(e));
  }
  cudaError_t e = cudaMemcpyAsync(status_host, status_dev, sizeof(int32_t) * b, cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor_solve_host: D2H %s", cudaGetErrorString(e));
  return RR_OK;
}


rr_err rr_factor_solve_host_pipelined(const rr_dims* dims, const rr_problem* ph, const rr_solution* sh,
                                      int32_t* status_host, const rr_problem* pd, const rr_solution* sd,
                                      int32_t* status_dev, void* workspace, int64_t workspace_bytes, int32_t nchunks,
                                      void* const* streams, int32_t nstreams) {
  if (!dims_ok(dims)) return set_err(RR_E_INVALID, "rr_factor_solve_host_pipelined: invalid dims%s");
  if (!ph || !sh || !pd || !sd || !status_host || !status_dev || !streams || nstreams < 1 || nchunks < 1)
    return set_err(RR_E_INVALID, "rr_factor_solve_host_pipelined: null or invalid %s", "argument");
  if (dims->batch == 0) return RR_OK;
  const int64_t b = dims->batch, N = dims->N, n = dims->nx, m = dims->nu;
  const int64_t sn = n * (n + 1) / 2, sm = m * (m + 1) / 2;
  const bool shD = (dims->flags & RR_FLAG_SHARED_DYN) != 0, shP = (dims->flags & RR_FLAG_SHARED_COST) != 0;
  const int64_t nD = (dims->flags & RR_FLAG_STAGE_INVARIANT_DYN) ? 1 : N;   // stage blocks of A, B
  const int64_t nP = (dims->flags & RR_FLAG_STAGE_INVARIANT_COST) ? 1 : N;  // stage blocks of Q, M, R
  const int64_t nc = nchunks > b ? b : nchunks;
  // per-chunk workspace slices, each 256-byte aligned, carved from the caller's buffer
  int64_t need = 0;
  for (int64_t c = 0; c < nc; ++c) {
    rr_dims dc = *dims;
    dc.batch = b * (c + 1) / nc - b * c / nc;
    const int64_t w = rr_workspace_bytes(&dc);
    if (w < 0) return set_err(RR_E_UNSUPPORTED, "rr_factor_solve_host_pipelined: no kernel for this shape%s");
    need += (w + 255) & ~(int64_t)255;
  }
  if (workspace == nullptr || workspace_bytes < need)
    return set_err(RR_E_INVALID, "rr_factor_solve_host_pipelined: workspace smaller than %s",
                   "the sum of rr_workspace_bytes over the chunks (+256 B alignment each)");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0)
    return set_err(RR_E_INVALID, "rr_factor_solve_host_pipelined: workspace not %s", "256-byte aligned");
  cudaStream_t s0 = static_cast<cudaStream_t>(streams[0]);
  auto h2d = [&](const double* h, const double* d, int64_t off, int64_t cnt, cudaStream_t s) -> cudaError_t {
    if (cnt == 0) return cudaSuccess;
    if (!h || !d) return cudaErrorInvalidValue;
    return cudaMemcpyAsync(const_cast<double*>(d) + off, h + off, sizeof(double) * cnt, cudaMemcpyHostToDevice, s);
  };
  cudaError_t e = cudaSuccess;
  // batch-shared operands once, on streams[0], before the fork
  if (shD) {
    if ((e = h2d(ph->A, pd->A, 0, nD * n * n, s0)) != cudaSuccess || (e = h2d(ph->B, pd->B, 0, nD * n * m, s0)) != cudaSuccess)
      return set_err(RR_E_CUDA, "rr_factor_solve_host_pipelined: H2D %s", cudaGetErrorString(e));
  }
  if (shP) {
    if ((e = h2d(ph->Q, pd->Q, 0, nP * sn, s0)) != cudaSuccess || (e = h2d(ph->M, pd->M, 0, nP * n * m, s0)) != cudaSuccess ||
        (e = h2d(ph->R, pd->R, 0, nP * sm, s0)) != cudaSuccess || (e = h2d(ph->QN, pd->QN, 0, sn, s0)) != cudaSuccess)
      return set_err(RR_E_CUDA, "rr_factor_solve_host_pipelined: H2D %s", cudaGetErrorString(e));
  }
  // fork: streams[1..] wait for everything enqueued on streams[0] so far
  cudaEvent_t fork = nullptr;
  if (nstreams > 1) {
    if ((e = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventRecord(fork, s0)) != cudaSuccess)
      return set_err(RR_E_CUDA, "rr_factor_solve_host_pipelined: event %s", cudaGetErrorString(e));
    for (int k = 1; k < nstreams; ++k)
      if ((e = cudaStreamWaitEvent(static_cast<cudaStream_t>(streams[k]), fork, 0)) != cudaSuccess) break;
    cudaEventDestroy(fork);  // released once the recorded work completes
    if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor_solve_host_pipelined: event %s", cudaGetErrorString(e));
  }
  char* wsp = static_cast<char*>(workspace);
  for (int64_t c = 0; c < nc && e == cudaSuccess; ++c) {
    cudaStream_t s = static_cast<cudaStream_t>(streams[c % nstreams]);
    const int64_t i0 = b * c / nc, cb = b * (c + 1) / nc - i0;
    rr_dims dc = *dims;
    dc.batch = cb;
    // H2D of the chunk's slices (every per-instance operand is [batch][...] contiguous)
    struct Op { const double* h; const double* d; int64_t per; bool inst; } ops[] = {
        {ph->A, pd->A, nD * n * n, !shD}, {ph->B, pd->B, nD * n * m, !shD}, {ph->Q, pd->Q, nP * sn, !shP},
        {ph->M, pd->M, nP * n * m, !shP}, {ph->R, pd->R, nP * sm, !shP},    {ph->q, pd->q, N * n, true},
        {ph->r, pd->r, N * m, true},     {ph->c, pd->c, N * n, true},     {ph->QN, pd->QN, sn, !shP},
        {ph->qN, pd->qN, n, true},       {ph->c0, pd->c0, n, true},       {ph->delta, pd->delta, 1, true}};
    for (const Op& o : ops)
      if (o.inst && (e = h2d(o.h, o.d, i0 * o.per, cb * o.per, s)) != cudaSuccess) break;
    if (e != cudaSuccess) break;
    // the chunk's problem / solution views (batch-shared operands keep their base pointers)
    rr_problem pc = *pd;
    auto off = [&](const double* p, int64_t per, bool inst) { return (inst && p) ? p + i0 * per : p; };
    pc.A = off(pd->A, nD * n * n, !shD);
    pc.B = off(pd->B, nD * n * m, !shD);
    pc.Q = off(pd->Q, nP * sn, !shP);
    pc.M = off(pd->M, nP * n * m, !shP);
    pc.R = off(pd->R, nP * sm, !shP);
    pc.q = off(pd->q, N * n, true);
    pc.r = off(pd->r, N * m, true);
    pc.c = off(pd->c, N * n, true);
    pc.QN = off(pd->QN, sn, !shP);
    pc.qN = off(pd->qN, n, true);
    pc.c0 = off(pd->c0, n, true);
    pc.delta = off(pd->delta, 1, true);
    rr_solution sc = {sd->x + i0 * (N + 1) * n, sd->u ? sd->u + i0 * N * m : nullptr, sd->y + i0 * (N + 1) * n};
    const int64_t wb = rr_workspace_bytes(&dc);
    rr_err rc = rr_factor_solve(&dc, &pc, nullptr, &sc, wsp, wb, status_dev + i0, s);
    if (rc != RR_OK) return rc;
    wsp += (wb + 255) & ~(int64_t)255;
    struct Out { double* h; const double* d; int64_t per; } outs[] = {
        {sh->x, sd->x, (N + 1) * n}, {sh->u, sd->u, N * m}, {sh->y, sd->y, (N + 1) * n}};
    for (const Out& o : outs) {
      if (o.per == 0 || o.h == nullptr) continue;
      if ((e = cudaMemcpyAsync(o.h + i0 * o.per, o.d + i0 * o.per, sizeof(double) * cb * o.per, cudaMemcpyDeviceToHost,
                               s)) != cudaSuccess)
        break;
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(status_host + i0, status_dev + i0, sizeof(int32_t) * cb, cudaMemcpyDeviceToHost, s);
  }
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor_solve_host_pipelined: copy %s", cudaGetErrorString(e));
  // join: streams[0] waits for the others, so its completion is the call's completion
  for (int k = 1; k < nstreams; ++k) {
    cudaEvent_t join = nullptr;
    if ((e = cudaEventCreateWithFlags(&join, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventRecord(join, static_cast<cudaStream_t>(streams[k]))) != cudaSuccess ||
        (e = cudaStreamWaitEvent(s0, join, 0)) != cudaSuccess) {
      if (join) cudaEventDestroy(join);
      return set_err(RR_E_CUDA, "rr_factor_solve_host_pipelined: event %s", cudaGetErrorString(e));
    }
    cudaEventDestroy(join);
  }
  return RR_OK;
}

int32_t rr_factor_record_doubles(int32_t n, int32_t m) { return rrk::frec_doubles(n, m); }

int64_t rr_factor_bytes(const rr_dims* dims) {
  if (!dims_ok(dims, RR_FLAG_ACCUMULATE | SHARED_FLAGS | RR_FLAG_FACTOR_FP32) || !rrk::split_supported(dims->nx, dims->nu))
    return -1;
  if (dims->flags & RR_FLAG_FACTOR_FP32) {  // FP32 records: the 12x4 DMMA factor kernel and rr_solve<12,4>
    if (dims->nx != 12 || dims->nu != 4) return -1;
    return dims->batch * (int64_t)(dims->N + 1) * rrk::frec_floats(dims->nx, dims->nu) * 4;
  }
  return dims->batch * (int64_t)(dims->N + 1) * rrk::frec_doubles(dims->nx, dims->nu) * 8;
}

int64_t rr_solve_workspace_bytes(const rr_dims* dims) {
  if (!dims_ok(dims, RR_FLAG_ACCUMULATE | SHARED_FLAGS | RR_FLAG_FACTOR_FP32) || !rrk::split_supported(dims->nx, dims->nu))
    return -1;
  return dims->batch * (int64_t)dims->N * (dims->nx + dims->nu) * 8 + 256;
}

rr_err rr_factor(const rr_dims* dims, const rr_problem* prob, void* factor, int64_t factor_bytes,
                 const rr_factor_buf* fac, int32_t* status, void* stream) {
  if (!dims_ok(dims, SHARED_FLAGS | RR_FLAG_FACTOR_FP32)) return set_err(RR_E_INVALID, "rr_factor: invalid dims%s");
  if (prob == nullptr) return set_err(RR_E_INVALID, "rr_factor: null %s", "prob");
  if (dims->batch == 0) return RR_OK;
  if (status == nullptr) return set_err(RR_E_INVALID, "rr_factor: null %s", "status");
  if (prob->QN == nullptr || prob->delta == nullptr)
    return set_err(RR_E_INVALID, "rr_factor: null %s", "QN/delta");
  if (dims->N > 0) {
    const double* req[] = {prob->A, prob->B, prob->Q, prob->M, prob->R};
    for (const double* p : req)
      if (p == nullptr) return set_err(RR_E_INVALID, "rr_factor: null %s", "stage operand (A, B, Q, M, R)");
  }
  const int64_t need = rr_factor_bytes(dims);
  if (need < 0) return set_err(RR_E_UNSUPPORTED, "rr_factor: no kernel compiled for this (nx, nu)%s");
  if (factor == nullptr || factor_bytes < need)
    return set_err(RR_E_INVALID, "rr_factor: factor buffer missing or smaller than %s", "rr_factor_bytes()");
  if ((reinterpret_cast<uintptr_t>(factor) & 15u) != 0)
    return set_err(RR_E_INVALID, "rr_factor: factor buffer not %s", "16-byte aligned");
  rrk::SplitArgs a{};
  a.nx = dims->nx;
  a.nu = dims->nu;
  a.N = dims->N;
  a.batch = dims->batch;
  a.p = *prob;
  rr_factor_buf none = {nullptr, nullptr, nullptr, nullptr};
  a.f = fac ? *fac : none;
  a.f.v = nullptr;
  a.f.k = nullptr;
  a.fr = static_cast<double*>(factor);
  a.status = status;
  a.shared = dims->flags & SHARED_FLAGS;
  a.tma16 = stage_ops_aligned16(prob);
  a.f32 = (dims->flags & RR_FLAG_FACTOR_FP32) != 0;
  if (a.f32 && !a.tma16)
    return set_err(RR_E_UNSUPPORTED, "rr_factor: FP32 records need 16-byte aligned stage operands%s");
  bool supported = false;
  cudaError_t e = rrk::factor_launch(a, static_cast<cudaStream_t>(stream), &supported);
  if (!supported) return set_err(RR_E_UNSUPPORTED, "rr_factor: unsupported shape%s");
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

rr_err rr_solve(const rr_dims* dims, const rr_problem* prob, const void* factor, int64_t factor_bytes,
                const rr_factor_buf* fac, const rr_solution* sol, void* workspace, int64_t workspace_bytes,
                int32_t* status, void* stream) {
  if (!dims_ok(dims, RR_FLAG_ACCUMULATE | SHARED_FLAGS | RR_FLAG_FACTOR_FP32))
    return set_err(RR_E_INVALID, "rr_solve: invalid dims%s");
  if (prob == nullptr || sol == nullptr) return set_err(RR_E_INVALID, "rr_solve: null %s", "prob/sol");
  if (dims->batch == 0) return RR_OK;
  if (status == nullptr) return set_err(RR_E_INVALID, "rr_solve: null %s", "status");
  if (prob->qN == nullptr || prob->c0 == nullptr || prob->delta == nullptr)
    return set_err(RR_E_INVALID, "rr_solve: null %s", "qN/c0/delta");
  if (dims->N > 0) {
    const double* req[] = {prob->A, prob->B, prob->q, prob->r, prob->c};
    for (const double* p : req)
      if (p == nullptr) return set_err(RR_E_INVALID, "rr_solve: null %s", "stage operand (A, B, q, r, c)");
  }
  if (sol->x == nullptr || sol->y == nullptr || (dims->N > 0 && sol->u == nullptr))
    return set_err(RR_E_INVALID, "rr_solve: null %s", "solution pointer");
  const int64_t need_f = rr_factor_bytes(dims), need_w = rr_solve_workspace_bytes(dims);
  if (need_f < 0 || need_w < 0) return set_err(RR_E_UNSUPPORTED, "rr_solve: no kernel compiled for this (nx, nu)%s");
  if (factor == nullptr || factor_bytes < need_f)
    return set_err(RR_E_INVALID, "rr_solve: factor buffer missing or smaller than %s", "rr_factor_bytes()");
  if ((reinterpret_cast<uintptr_t>(factor) & 15u) != 0)
    return set_err(RR_E_INVALID, "rr_solve: factor buffer not %s", "16-byte aligned");
  if (dims->N > 0 && (workspace == nullptr || workspace_bytes < need_w))
    return set_err(RR_E_INVALID, "rr_solve: workspace missing or smaller than %s", "rr_solve_workspace_bytes()");
  rrk::SplitArgs a{};
  a.nx = dims->nx;
  a.nu = dims->nu;
  a.N = dims->N;
  a.batch = dims->batch;
  a.p = *prob;
  rr_factor_buf none = {nullptr, nullptr, nullptr, nullptr};
  a.f = fac ? *fac : none;
  a.f.V = nullptr;
  a.f.K = nullptr;
  a.s = *sol;
  a.frc = static_cast<const double*>(factor);
  a.ws = static_cast<double*>(workspace);
  a.status = status;
  a.accumulate = (dims->flags & RR_FLAG_ACCUMULATE) != 0;
  a.shared = dims->flags & SHARED_FLAGS;
  a.f32 = (dims->flags & RR_FLAG_FACTOR_FP32) != 0;
  bool supported = false;
  cudaError_t e = rrk::solve_launch(a, static_cast<cudaStream_t>(stream), &supported);
  if (!supported) return set_err(RR_E_UNSUPPORTED, "rr_solve: unsupported shape%s");
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_solve: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

rr_err rr_residual(const rr_dims* dims, const rr_problem* prob, const rr_solution* sol, const rr_residual_buf* res,
                   double* norms, void* stream) {
  if (!dims_ok(dims)) return set_err(RR_E_INVALID, "rr_residual: invalid dims%s");
  if (prob == nullptr || sol == nullptr) return set_err(RR_E_INVALID, "rr_residual: null %s", "prob/sol");
  if (dims->batch == 0) return RR_OK;
  const double* req[] = {prob->QN, prob->qN, prob->c0, prob->delta, sol->x, sol->y};
  for (const double* p : req)
    if (p == nullptr) return set_err(RR_E_INVALID, "rr_residual: null %s", "terminal operand or solution");
  if (dims->N > 0) {
    const double* req2[] = {prob->A, prob->B, prob->Q, prob->M, prob->R, prob->q, prob->r, prob->c, sol->u};
    for (const double* p : req2)
      if (p == nullptr) return set_err(RR_E_INVALID, "rr_residual: null %s", "stage operand or u");
  }
  if (!rrk::split_supported(dims->nx, dims->nu))
    return set_err(RR_E_UNSUPPORTED, "rr_residual: no kernel compiled for this (nx, nu)%s");
  rrk::ResArgs a{};
  a.nx = dims->nx;
  a.nu = dims->nu;
  a.N = dims->N;
  a.batch = dims->batch;
  a.p = *prob;
  a.s = *sol;
  rr_residual_buf none = {nullptr, nullptr, nullptr, nullptr, nullptr};
  a.r = res ? *res : none;
  a.norms = norms;
  a.shared = dims->flags & SHARED_FLAGS;
  bool supported = false;
  cudaError_t e = rrk::residual_launch(a, static_cast<cudaStream_t>(stream), &supported);
  if (!supported) return set_err(RR_E_UNSUPPORTED, "rr_residual: unsupported shape%s");
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_residual: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

int64_t rr_pit_workspace_bytes(const rr_dims* dims) {
  if (!dims_ok(dims)) return -1;
  return rrk::pit_ws_bytes(dims->nx, dims->nu, dims->N, dims->batch);
}

rr_err rr_factor_solve_pit(const rr_dims* dims, const rr_problem* prob, const rr_solution* sol, void* workspace,
                           int64_t workspace_bytes, int32_t* status, void* stream) {
  if (!dims_ok(dims)) return set_err(RR_E_INVALID, "rr_factor_solve_pit: invalid dims%s");
  if (prob == nullptr || sol == nullptr) return set_err(RR_E_INVALID, "rr_factor_solve_pit: null %s", "prob/sol");
  if (dims->batch == 0) return RR_OK;
  if (status == nullptr) return set_err(RR_E_INVALID, "rr_factor_solve_pit: null %s", "status");
  const double* req[] = {prob->QN, prob->qN, prob->c0, prob->delta, sol->x, sol->y};
  for (const double* p : req)
    if (p == nullptr) return set_err(RR_E_INVALID, "rr_factor_solve_pit: null %s", "terminal operand / solution");
  if (dims->N > 0) {
    const double* req2[] = {prob->A, prob->B, prob->Q, prob->M, prob->R, prob->q, prob->r, prob->c, sol->u};
    for (const double* p : req2)
      if (p == nullptr) return set_err(RR_E_INVALID, "rr_factor_solve_pit: null %s", "stage operand / u");
  }
  const int64_t need = rr_pit_workspace_bytes(dims);
  if (need < 0) return set_err(RR_E_UNSUPPORTED, "rr_factor_solve_pit: nx, nu must be <= 16%s");
  if (workspace == nullptr || workspace_bytes < need)
    return set_err(RR_E_INVALID, "rr_factor_solve_pit: workspace missing or smaller than %s", "rr_pit_workspace_bytes()");
  rrk::PitArgs a{};
  a.nx = dims->nx;
  a.nu = dims->nu;
  a.N = dims->N;
  a.batch = dims->batch;
  a.p = *prob;
  a.s = *sol;
  a.ws = static_cast<double*>(workspace);
  a.status = status;
  a.shared = dims->flags & SHARED_FLAGS;
  // reduction at δ_s = max(δ, 1e-4), then 2 refinement steps on the caller's δ (δ = 0 included):
  // measured 1e-8 -> 1e-12 -> 1e-16 relative error on C2-shaped and C4-shaped instances at δ = 0
  a.delta_floor = 1e-4;
  a.refine = 2;
  if (const char* v = getenv("RR_PIT_REFINE")) a.refine = atoi(v);           // A/B knobs
  if (const char* v = getenv("RR_PIT_DELTA_FLOOR")) a.delta_floor = atof(v);
  cudaError_t e = rrk::pit_launch(a, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "rr_factor_solve_pit: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

static bool ipm_dims_ok(const ipm_dims* d) {
  return d != nullptr && d->nx >= 1 && d->nu >= 1 && d->N >= 0 && d->batch >= 0 && d->ng >= 0 && d->ngN >= 0 &&
         d->nc >= 0 && d->ncN >= 0 && (d->model == IPM_MODEL_LQ || d->model == IPM_MODEL_CARTPOLE || d->model == IPM_MODEL_QUADROTOR);
}

int64_t ipm_workspace_bytes(const ipm_dims* dims) {
  if (!ipm_dims_ok(dims)) return -1;
  return rrk::ipm_ws_bytes(*dims);
}

static rr_err ipm_step_impl(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it,
                            const ipm_params* params, const ipm_result* res, void* workspace, int64_t workspace_bytes,
                            int32_t* status, void* stream, int direction_only);

rr_err ipm_step(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it, const ipm_params* params,
                const ipm_result* res, void* workspace, int64_t workspace_bytes, int32_t* status, void* stream) {
  return ipm_step_impl(dims, data, it, params, res, workspace, workspace_bytes, status, stream, 0);
}

rr_err ipm_direction(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it, const ipm_params* params,
                     const ipm_result* res, void* workspace, int64_t workspace_bytes, int32_t* status, void* stream) {
  return ipm_step_impl(dims, data, it, params, res, workspace, workspace_bytes, status, stream, 1);
}

// Arrays a dimension makes required (include/rr.h ipm_* structs): stage data and iterate/result
// blocks of every non-empty dimension must be non-NULL (the kernels index them unconditionally).
static bool ipm_iterate_ok(const ipm_dims* d, const ipm_iterate* it) {
  if (!it->x || !it->y || !it->mu || !it->eta) return false;
  if (d->N > 0 && !it->u) return false;
  if (d->N > 0 && d->ng > 0 && (!it->s || !it->z)) return false;
  if (d->ngN > 0 && (!it->sN || !it->zN)) return false;
  if (d->N > 0 && d->nc > 0 && !it->lam) return false;
  if (d->ncN > 0 && !it->lamN) return false;
  return true;
}
static bool ipm_direction_ok(const ipm_dims* d, const ipm_result* r) {
  if (!r->dx || !r->dy) return false;
  if (d->N > 0 && !r->du) return false;
  if (d->N > 0 && d->ng > 0 && (!r->ds || !r->dz)) return false;
  if (d->ngN > 0 && (!r->dsN || !r->dzN)) return false;
  if (d->N > 0 && d->nc > 0 && !r->dlam) return false;
  if (d->ncN > 0 && !r->dlamN) return false;
  return true;
}
static bool ipm_data_ok(const ipm_dims* d, const ipm_stage_data* D) {
  if (!D->s0 || !D->fval || !D->gradfN || !D->QN) return false;
  if (d->N > 0 && (!D->gradf || !D->Q || !D->M || !D->R || !D->A || !D->B || !D->dres)) return false;
  if (d->N > 0 && d->ng > 0 && (!D->gv || !D->Gj)) return false;
  if (d->ngN > 0 && (!D->gvN || !D->GjN)) return false;
  if (d->N > 0 && d->nc > 0 && (!D->ce || !D->Ce)) return false;
  if (d->ncN > 0 && (!D->ceN || !D->CeN)) return false;
  return true;
}

rr_err ipm_merit(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it, const ipm_result* res,
                 const double* alpha, const ipm_trial_values* trial, double* merit, void* stream) {
  if (!ipm_dims_ok(dims)) return set_err(RR_E_INVALID, "ipm_merit: invalid dims%s");
  if (!data || !it || !res || !trial) return set_err(RR_E_INVALID, "ipm_merit: null %s", "argument");
  if (dims->batch == 0) return RR_OK;
  if (!alpha || !merit || !trial->fval || !data->s0 || !it->x || !it->y || !it->mu || !it->eta || !res->dx ||
      (dims->N > 0 && !trial->dres) || (dims->ng > 0 && (!trial->gv || !it->s || !it->z || !res->ds)) ||
      (dims->ngN > 0 && (!trial->gvN || !it->sN || !it->zN || !res->dsN)) || (dims->nc > 0 && (!trial->ce || !it->lam)) ||
      (dims->ncN > 0 && (!trial->ceN || !it->lamN)))
    return set_err(RR_E_INVALID, "ipm_merit: null %s", "required pointer");
  cudaError_t e = rrk::ipm_merit_launch(*dims, *data, *it, *res, alpha, *trial, merit, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "ipm_merit: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

rr_err ipm_update(const ipm_dims* dims, const ipm_iterate* it, const ipm_result* res, const double* alpha_p,
                  const double* alpha_d, void* stream) {
  if (!ipm_dims_ok(dims)) return set_err(RR_E_INVALID, "ipm_update: invalid dims%s");
  if (!it || !res) return set_err(RR_E_INVALID, "ipm_update: null %s", "argument");
  if (dims->batch == 0) return RR_OK;
  if (!alpha_p || !alpha_d || !ipm_iterate_ok(dims, it) || !ipm_direction_ok(dims, res))
    return set_err(RR_E_INVALID, "ipm_update: null %s", "required pointer (iterate or direction block of a non-empty dimension)");
  cudaError_t e = rrk::ipm_update_launch(*dims, *it, *res, alpha_p, alpha_d, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "ipm_update: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

static rr_err ipm_step_impl(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it,
                            const ipm_params* params, const ipm_result* res, void* workspace, int64_t workspace_bytes,
                            int32_t* status, void* stream, int direction_only) {
  if (!ipm_dims_ok(dims)) return set_err(RR_E_INVALID, "ipm_step: invalid dims%s");
  if (!data || !it || !params || !res) return set_err(RR_E_INVALID, "ipm_step: null %s", "argument");
  if (dims->batch == 0) return RR_OK;  // nothing to do; status may be null for an empty batch
  if (!status) return set_err(RR_E_INVALID, "ipm_step: null %s", "status");
  if (!(params->tau > 0.0 && params->tau < 1.0) || !(params->armijo_c > 0.0 && params->armijo_c < 0.5) ||
      !(params->beta > 0.0 && params->beta < 1.0) || params->max_backtracks < 0)
    return set_err(RR_E_INVALID, "ipm_step: invalid %s", "line-search parameters");
  const int64_t need = ipm_workspace_bytes(dims);
  if (need < 0) return set_err(RR_E_UNSUPPORTED, "ipm_step: no kernel compiled for these dims/model%s");
  if (dims->N > 0 && (workspace == nullptr || workspace_bytes < need))
    return set_err(RR_E_INVALID, "ipm_step: workspace missing or smaller than %s", "ipm_workspace_bytes()");
  if (!ipm_data_ok(dims, data) || !ipm_iterate_ok(dims, it) || !ipm_direction_ok(dims, res))
    return set_err(RR_E_INVALID, "ipm_step: null %s", "required pointer (data, iterate or direction block of a non-empty dimension)");
  if (dims->model != IPM_MODEL_LQ && data->model_params == nullptr)
    return set_err(RR_E_INVALID, "ipm_step: the built-in nonlinear models need %s", "model_params");
  rrk::IpmArgs a;
  a.d = *dims;
  a.d_ = *data;
  a.it = *it;
  a.prm = *params;
  a.r = *res;
  a.ws = static_cast<double*>(workspace);
  a.status = status;
  a.direction_only = direction_only;
  bool supported = false;
  cudaError_t e = rrk::ipm_launch(a, static_cast<cudaStream_t>(stream), &supported);
  if (!supported) return set_err(RR_E_UNSUPPORTED, "ipm_step: unsupported dims%s");
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "ipm_step: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

int64_t ipm_solve_workspace_bytes(const ipm_dims* dims) {
  if (!ipm_dims_ok(dims)) return -1;
  return rrk::ipm_solve_ws_bytes(*dims);
}

rr_err ipm_solve(const ipm_dims* dims, const ipm_stage_data* data, const ipm_iterate* it,
                 const ipm_solve_settings* S, const ipm_solve_report* rep, void* workspace, int64_t workspace_bytes,
                 void* stream) {
  if (!ipm_dims_ok(dims)) return set_err(RR_E_INVALID, "ipm_solve: invalid dims%s");
  if (!data || !it || !S || !rep) return set_err(RR_E_INVALID, "ipm_solve: null %s", "argument");
  if (dims->batch == 0) return RR_OK;
  const ipm_params& p = S->step;
  if (!(p.tau > 0.0 && p.tau < 1.0) || !(p.armijo_c > 0.0 && p.armijo_c < 0.5) || !(p.beta > 0.0 && p.beta < 1.0) ||
      p.max_backtracks < 0 || S->max_iters < 0 || !(S->mu_min > 0.0) || !(S->kappa_mu > 0.0 && S->kappa_mu < 1.0) ||
      !(S->theta_mu > 1.0) || !(S->tol_kkt > 0.0) || !(S->kappa > 0.0) || !(S->kappa_eta >= 1.0) || !(S->eta_max > 0.0))
    return set_err(RR_E_INVALID, "ipm_solve: invalid %s", "settings");
  if (dims->batch > 0x7fffffffLL) return set_err(RR_E_INVALID, "ipm_solve: batch above %s", "2^31-1");
  const int64_t need = ipm_solve_workspace_bytes(dims);
  if (need < 0) return set_err(RR_E_UNSUPPORTED, "ipm_solve: no kernel compiled for these dims/model%s");
  if (workspace == nullptr || workspace_bytes < need)
    return set_err(RR_E_INVALID, "ipm_solve: workspace missing or smaller than %s", "ipm_solve_workspace_bytes()");
  if (!ipm_data_ok(dims, data) || !ipm_iterate_ok(dims, it))
    return set_err(RR_E_INVALID, "ipm_solve: null %s", "required pointer (data or iterate block of a non-empty dimension)");
  if (dims->model != IPM_MODEL_LQ && data->model_params == nullptr)
    return set_err(RR_E_INVALID, "ipm_solve: the built-in nonlinear models need %s", "model_params");
  bool supported = false;
  cudaError_t e = rrk::ipm_solve_launch(*dims, *data, *it, *S, *rep, workspace, static_cast<cudaStream_t>(stream),
                                        &supported);
  if (!supported) return set_err(RR_E_UNSUPPORTED, "ipm_solve: unsupported dims%s");
  if (e != cudaSuccess) return set_err(RR_E_CUDA, "ipm_solve: CUDA error %s", cudaGetErrorString(e));
  return RR_OK;
}

}  // extern "C"
