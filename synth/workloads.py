"""Seeded synthetic workloads (inputs only) for the regularized-LQR hot path.

This module is shared by the CUDA path's tests/bench and by the oracle's tests.
It holds NONE of the method's arithmetic (no Riccati step, no factorization, no
IPM elimination): it only draws random numbers and assembles input matrices with
the definiteness the paper requires of them (§1.4: P_i PSD, R_i PD).

Random numbers come from a counter-based generator (SplitMix64 over
(seed, global instance id, stage, operand, element)), written with torch int64
ops so that the same integer stream is produced on CPU and on CUDA, and so an
instance's inputs depend only on its global id (sharding-invariant).

Layout (the C-ABI layout, include/rr.h): one tensor per operand, shaped
[batch, N, elems] (or [batch, elems] for terminal data), matrices column-major
and flattened, symmetric matrices packed lower (LAPACK 'L' packed order).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, Optional

import torch

# operand ids for the counter (part of the workload definition)
OP_A, OP_B, OP_L, OP_Q, OP_R, OP_C, OP_QN, OP_QNV, OP_C0 = range(9)

_M1 = 0x9E3779B97F4A7C15
_M2 = 0xBF58476D1CE4E5B9
_M3 = 0x94D049BB133111EB


def _s64(v: int) -> int:
    """Unsigned 64-bit constant -> the signed int64 with the same bits."""
    v &= (1 << 64) - 1
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    """Logical right shift of int64 bit patterns."""
    return torch.bitwise_and(torch.bitwise_right_shift(z, s), (1 << (64 - s)) - 1)


def splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _s64(_M1)
    z = torch.bitwise_xor(z, _lsr(z, 30)) * _s64(_M2)
    z = torch.bitwise_xor(z, _lsr(z, 27)) * _s64(_M3)
    return torch.bitwise_xor(z, _lsr(z, 31))


def uniform(seed: int, inst: torch.Tensor, stage: int | torch.Tensor, operand: int, nelem: int,
            device=None) -> torch.Tensor:
    """U(-1,1) doubles for every (instance in `inst`, stage, element < nelem).

    inst: int64 tensor [b] of global instance ids; stage: int or int64 tensor [S].
    Returns [b, S, nelem] (or [b, nelem] when stage is an int)."""
    device = inst.device if device is None else device
    scalar_stage = isinstance(stage, int)
    st = torch.tensor([stage], dtype=torch.int64, device=device) if scalar_stage else stage.to(device)
    e = torch.arange(nelem, dtype=torch.int64, device=device)
    # counter = (((inst * 2^12 + stage) * 2^4 + operand) * 2^16 + elem)  -- unique for
    # inst < 2^31, stage < 2^12, operand < 16, elem < 2^16
    ctr = ((inst.view(-1, 1, 1) * 4096 + st.view(1, -1, 1)) * 16 + operand) * 65536 + e.view(1, 1, -1)
    z = splitmix64(ctr ^ splitmix64(torch.tensor(seed, dtype=torch.int64, device=device)))
    u = _lsr(z, 11).to(torch.float64) * (1.0 / 9007199254740992.0)
    out = 2.0 * u - 1.0
    return out[:, 0, :] if scalar_stage else out


def sym_size(n: int) -> int:
    return n * (n + 1) // 2


def pack_lower(F: torch.Tensor) -> torch.Tensor:
    """[..., n, n] (F[..., r, c]) -> [..., sym(n)] in LAPACK 'L' packed column order."""
    n = F.shape[-1]
    rows, cols = [], []
    for c in range(n):
        for r in range(c, n):
            rows.append(r)
            cols.append(c)
    return F[..., rows, cols]


def unpack_lower(P: torch.Tensor, n: int) -> torch.Tensor:
    """[..., sym(n)] -> symmetric [..., n, n]."""
    out = torch.zeros(P.shape[:-1] + (n, n), dtype=P.dtype, device=P.device)
    k = 0
    for c in range(n):
        for r in range(c, n):
            out[..., r, c] = P[..., k]
            out[..., c, r] = P[..., k]
            k += 1
    return out


def colmajor(F: torch.Tensor) -> torch.Tensor:
    """[..., r, c] -> flattened column-major [..., r*c]."""
    return F.transpose(-1, -2).reshape(F.shape[:-2] + (F.shape[-1] * F.shape[-2],))


def from_colmajor(f: torch.Tensor, rows: int, cols: int) -> torch.Tensor:
    return f.reshape(f.shape[:-1] + (cols, rows)).transpose(-1, -2)


@dataclasses.dataclass
class RRProblem:
    """A batch of regularized LQR instances in the C-ABI layout."""
    nx: int
    nu: int
    N: int
    A: torch.Tensor      # [b, N, nx*nx]
    B: torch.Tensor      # [b, N, nx*nu]
    Q: torch.Tensor      # [b, N, sym(nx)]
    M: torch.Tensor      # [b, N, nx*nu]
    R: torch.Tensor      # [b, N, sym(nu)]
    q: torch.Tensor      # [b, N, nx]
    r: torch.Tensor      # [b, N, nu]
    c: torch.Tensor      # [b, N, nx]   c[:, i] = c_{i+1}
    QN: torch.Tensor     # [b, sym(nx)]
    qN: torch.Tensor     # [b, nx]
    c0: torch.Tensor     # [b, nx]
    delta: torch.Tensor  # [b]

    FIELDS = ("A", "B", "Q", "M", "R", "q", "r", "c", "QN", "qN", "c0", "delta")

    @property
    def batch(self) -> int:
        return self.delta.shape[0]

    def to(self, device) -> "RRProblem":
        kw = {f: getattr(self, f).to(device) for f in self.FIELDS}
        return RRProblem(self.nx, self.nu, self.N, **kw)

    def select(self, idx) -> "RRProblem":
        kw = {f: getattr(self, f)[idx].contiguous() for f in self.FIELDS}
        return RRProblem(self.nx, self.nu, self.N, **kw)

    def contiguous(self) -> "RRProblem":
        kw = {f: getattr(self, f).contiguous() for f in self.FIELDS}
        return RRProblem(self.nx, self.nu, self.N, **kw)

    def nbytes(self) -> int:
        return sum(getattr(self, f).numel() * 8 for f in self.FIELDS)

    def expanded(self) -> "RRProblem":
        """Per-instance, per-stage copy of a problem with batch-shared (RR_FLAG_SHARED_*: A, B, Q, M, R
        of shape [N, elems], Q_N [elems]) and / or stage-invariant (RR_FLAG_STAGE_INVARIANT_*: stage
        dimension 1, i.e. [b, 1, elems] or [1, elems]) operands: broadcast to [b, N, elems]."""
        b = self.batch
        kw = {}
        for f in self.FIELDS:
            t = getattr(self, f)
            if f in ("A", "B", "Q", "M", "R"):
                if t.dim() == 2:
                    t = t.unsqueeze(0)
                t = t.expand(b, self.N, t.shape[-1])
            elif f == "QN" and t.dim() == 1:
                t = t.unsqueeze(0).expand(b, t.shape[0])
            kw[f] = t.contiguous()
        return RRProblem(self.nx, self.nu, self.N, **kw)

    def with_delta(self, delta: float) -> "RRProblem":
        kw = {f: getattr(self, f) for f in self.FIELDS}
        kw["delta"] = torch.full_like(self.delta, float(delta))
        return RRProblem(self.nx, self.nu, self.N, **kw)


def random_stable_lqr(nx: int, nu: int, N: int, batch: int, seed: int, delta: float = 1e-4,
                      first: int = 0, device="cpu", rho: float = 0.95) -> RRProblem:
    """C2/C3 recipe:
    A_i = rho * Ahat / ||Ahat||_F (Ahat ~ U(-1,1)), so ||A_i||_2 <= rho < 1;
    B_i ~ U(-1,1)/sqrt(nx);
    [[Q,M],[M^T,R]] = L L^T/(nx+nu) + blkdiag(0.1 I, I), L ~ U(-1,1)  (PSD P_i, PD R_i);
    Q_N = L_N L_N^T / nx + I;  q, r, c_0 ~ U(-1,1);  c_{i+1} ~ 0.1 U(-1,1);  delta per instance.
    Instances are `first .. first+batch-1` (global ids)."""
    dev = torch.device(device)
    inst = torch.arange(first, first + batch, dtype=torch.int64, device=dev)
    st = torch.arange(N, dtype=torch.int64, device=dev)
    n, m, k = nx, nu, nx + nu
    Ahat = uniform(seed, inst, st, OP_A, n * n)                     # col-major already (any order is iid)
    A = rho * Ahat / torch.linalg.vector_norm(Ahat, dim=-1, keepdim=True)
    B = uniform(seed, inst, st, OP_B, n * m) / math.sqrt(n)
    Lf = from_colmajor(uniform(seed, inst, st, OP_L, k * k), k, k)
    P = Lf @ Lf.transpose(-1, -2) / k
    P[..., :n, :n] += 0.1 * torch.eye(n, dtype=P.dtype, device=dev)
    P[..., n:, n:] += torch.eye(m, dtype=P.dtype, device=dev)
    Q = pack_lower(P[..., :n, :n])
    M = colmajor(P[..., :n, n:].contiguous())
    R = pack_lower(P[..., n:, n:])
    q = uniform(seed, inst, st, OP_Q, n)
    r = uniform(seed, inst, st, OP_R, m)
    c = 0.1 * uniform(seed, inst, st, OP_C, n)
    LN = from_colmajor(uniform(seed, inst, 0, OP_QN, n * n), n, n)
    QN = pack_lower(LN @ LN.transpose(-1, -2) / n + torch.eye(n, dtype=torch.float64, device=dev))
    qN = uniform(seed, inst, 0, OP_QNV, n)
    c0 = uniform(seed, inst, 0, OP_C0, n)
    d = torch.full((batch,), float(delta), dtype=torch.float64, device=dev)
    return RRProblem(nx, nu, N, A.contiguous(), B.contiguous(), Q.contiguous(), M.contiguous(),
                     R.contiguous(), q.contiguous(), r.contiguous(), c.contiguous(), QN.contiguous(),
                     qN.contiguous(), c0.contiguous(), d)


def lti_problem(nx: int, nu: int, N: int, batch: int, seed: int, delta: float = 1e-4, shared_dyn: bool = True,
                shared_cost: bool = True, device="cpu") -> RRProblem:
    """Fleet / LTI-MPC shaped batch: the matrices of one C2-recipe instance (global id
    0) shared by every instance (A, B and/or Q, M, R, Q_N without a batch dimension), per-instance
    right-hand sides q, r, c, q_N, c_0 and δ from instances 1..batch of the same generator."""
    base = random_stable_lqr(nx, nu, N, 1, seed, delta, first=0, device=device)
    rhs = random_stable_lqr(nx, nu, N, batch, seed, delta, first=1, device=device)
    kw = {f: getattr(rhs, f) for f in RRProblem.FIELDS}
    if shared_dyn:
        kw["A"], kw["B"] = base.A[0].contiguous(), base.B[0].contiguous()
    if shared_cost:
        kw["Q"], kw["M"], kw["R"], kw["QN"] = (base.Q[0].contiguous(), base.M[0].contiguous(),
                                               base.R[0].contiguous(), base.QN[0].contiguous())
    return RRProblem(nx, nu, N, **kw)


def lti_invariant_problem(nx: int, nu: int, N: int, batch: int, seed: int, delta: float = 1e-4,
                          shared: bool = False, device="cpu") -> RRProblem:
    """Time-invariant (LTI-MPC) batch (RR_FLAG_STAGE_INVARIANT_*): per instance ONE stage
    block of A, B, Q, M, R (the stage-0 blocks of the C2 recipe) used at every stage, stored with a
    stage dimension of 1 ([b, 1, elems]); shared=True: also batch-shared (one block for all, [1, elems];
    Q_N [elems]).  Right-hand sides q, r, c, q_N, c_0 and δ per instance and stage as in the C2 recipe."""
    base = random_stable_lqr(nx, nu, N, 1 if shared else batch, seed, delta, first=0, device=device)
    rhs = random_stable_lqr(nx, nu, N, batch, seed, delta, first=1, device=device)
    kw = {f: getattr(rhs, f) for f in RRProblem.FIELDS}
    for f in ("A", "B", "Q", "M", "R"):
        blk = getattr(base, f)[:, :1].contiguous()          # [b or 1, 1, elems]
        kw[f] = blk[0].contiguous() if shared else blk
    kw["QN"] = base.QN[0].contiguous() if shared else base.QN
    return RRProblem(nx, nu, N, **kw)


def random_stable_lqr_chunked(nx, nu, N, batch, seed, delta=1e-4, device="cpu", chunk=4096,
                              out: Optional[RRProblem] = None) -> RRProblem:
    """Same instances as random_stable_lqr, generated `chunk` instances at a time to bound
    temporary memory; writes into preallocated `out` if given."""
    if out is None:
        out = empty_problem(nx, nu, N, batch, device)
    for s in range(0, batch, chunk):
        e = min(batch, s + chunk)
        p = random_stable_lqr(nx, nu, N, e - s, seed, delta, first=s, device=device)
        for f in RRProblem.FIELDS:
            getattr(out, f)[s:e].copy_(getattr(p, f))
        del p
    return out


def empty_problem(nx, nu, N, batch, device="cpu", pin_memory=False) -> RRProblem:
    n, m = nx, nu
    kw = dict(dtype=torch.float64, device=device)
    if pin_memory:
        kw["pin_memory"] = True
    return RRProblem(nx, nu, N,
                     A=torch.empty(batch, N, n * n, **kw), B=torch.empty(batch, N, n * m, **kw),
                     Q=torch.empty(batch, N, sym_size(n), **kw), M=torch.empty(batch, N, n * m, **kw),
                     R=torch.empty(batch, N, sym_size(m), **kw), q=torch.empty(batch, N, n, **kw),
                     r=torch.empty(batch, N, m, **kw), c=torch.empty(batch, N, n, **kw),
                     QN=torch.empty(batch, sym_size(n), **kw), qN=torch.empty(batch, n, **kw),
                     c0=torch.empty(batch, n, **kw), delta=torch.empty(batch, **kw))


def double_integrator_c1(N: int = 10, h: float = 0.1, eta: float = 1e4,
                         s0=(5.0, 0.0)) -> RRProblem:
    """C1 (BASELINE configs[0]): double integrator A=[[1,h],[0,1]],
    B=[[h^2/2],[h]], Q=I, R=0.1, M=0, Q_N=10 I, linearised at xbar=0, ubar=0, so
    c_0 = s_0 - xbar_0 = s0 and c_{i+1} = 0, q = r = 0.  The terminal equality x_N[0] = 0
    is condensed per P:295-298 as Q_N += eta e1 e1^T (its residual is 0 at xbar), and
    delta = 1/eta."""
    n, m = 2, 1
    A = torch.tensor([[1.0, h], [0.0, 1.0]], dtype=torch.float64)
    B = torch.tensor([[h * h / 2], [h]], dtype=torch.float64)
    QN = 10.0 * torch.eye(2, dtype=torch.float64)
    QN[0, 0] += eta
    return RRProblem(
        n, m, N,
        A=colmajor(A).expand(1, N, 4).contiguous(), B=colmajor(B).expand(1, N, 2).contiguous(),
        Q=pack_lower(torch.eye(2, dtype=torch.float64)).expand(1, N, 3).contiguous(),
        M=torch.zeros(1, N, 2, dtype=torch.float64), R=torch.full((1, N, 1), 0.1, dtype=torch.float64),
        q=torch.zeros(1, N, 2, dtype=torch.float64), r=torch.zeros(1, N, 1, dtype=torch.float64),
        c=torch.zeros(1, N, 2, dtype=torch.float64), QN=pack_lower(QN).view(1, 3),
        qN=torch.zeros(1, 2, dtype=torch.float64), c0=torch.tensor([list(s0)], dtype=torch.float64),
        delta=torch.tensor([1.0 / eta], dtype=torch.float64))


def small_random(nx, nu, N, batch, seed, delta, psd_q=False, first=0) -> RRProblem:
    """Tiny instances for oracle pins (SPEC acceptance list S:498): like random_stable_lqr but
    optionally with a singular PSD Q (rank-deficient L L^T; P:379 allows PSD)."""
    p = random_stable_lqr(nx, nu, N, batch, seed, delta, first=first)
    if psd_q:
        n = nx
        inst = torch.arange(first, first + batch, dtype=torch.int64)
        st = torch.arange(N, dtype=torch.int64)
        v = uniform(seed + 1, inst, st, OP_Q, n)
        Qs = v.unsqueeze(-1) * v.unsqueeze(-2)          # rank one PSD
        p.Q = pack_lower(Qs).contiguous()
        p.M = torch.zeros_like(p.M)
    return p


# ----------------------------------------------------------------------------- C5 quadrotor
OP_XT, OP_UT, OP_XREF = 9, 10, 11


def quadrotor_f(x, u, mass=0.5, J=(2.32e-3, 2.32e-3, 4e-3), g=9.81):
    """Continuous quadrotor dynamics (workload definition): x = (p, ZYX Euler angles (φ, θ, ψ),
    world velocity, body rates ω), u = (thrust T, torques τ)."""
    phi, th, psi = x[..., 3], x[..., 4], x[..., 5]
    v = x[..., 6:9]
    w = x[..., 9:12]
    sph, cph, sth, cth, sps, cps = (torch.sin(phi), torch.cos(phi), torch.sin(th), torch.cos(th),
                                    torch.sin(psi), torch.cos(psi))
    # Euler-angle rates = W(φ, θ) ω
    dphi = w[..., 0] + sph * sth / cth * w[..., 1] + cph * sth / cth * w[..., 2]
    dth = cph * w[..., 1] - sph * w[..., 2]
    dpsi = sph / cth * w[..., 1] + cph / cth * w[..., 2]
    # world acceleration = R(φ, θ, ψ) [0, 0, T/m] − [0, 0, g]   (ZYX: R = Rz(ψ) Ry(θ) Rx(φ))
    T = u[..., 0]
    ax = (cps * sth * cph + sps * sph) * T / mass
    ay = (sps * sth * cph - cps * sph) * T / mass
    az = cth * cph * T / mass - g
    Jx, Jy, Jz = J
    tx, ty, tz = u[..., 1], u[..., 2], u[..., 3]
    dwx = (tx - (Jz - Jy) * w[..., 1] * w[..., 2]) / Jx
    dwy = (ty - (Jx - Jz) * w[..., 2] * w[..., 0]) / Jy
    dwz = (tz - (Jy - Jx) * w[..., 0] * w[..., 1]) / Jz
    return torch.stack([v[..., 0], v[..., 1], v[..., 2], dphi, dth, dpsi, ax, ay, az, dwx, dwy, dwz], dim=-1)


def quadrotor_c5(batch, seed=2512, N=200, first=0, device="cpu", dt=0.02, delta=1e-4) -> RRProblem:
    """C5 (BASELINE configs[4]): quadrotor LQR instances, n = 12, m = 4, N = 200.
    A_i = I + dt ∂f/∂x, B_i = dt ∂f/∂u (autograd) at random x̃ (p ~ U, angles ~ 0.3U, v ~ U,
    ω ~ 0.5U) and ũ = (m g (1 + 0.1U), 0.01U); Q = diag(10,10,10,1,1,1,1,1,1,.1,.1,.1),
    R = diag(0.1, 1, 1, 1), M = 0, Q_N = 10 Q, q = −Q x_ref (x_ref ~ U), r = 0, c ~ 0.01U,
    c_0 ~ U, δ = 1e-4."""
    dev = torch.device(device)
    n, m = 12, 4
    inst = torch.arange(first, first + batch, dtype=torch.int64, device=dev)
    st = torch.arange(N, dtype=torch.int64, device=dev)
    xs = uniform(seed, inst, st, OP_XT, n) * torch.tensor([1, 1, 1, .3, .3, .3, 1, 1, 1, .5, .5, .5],
                                                          dtype=torch.float64, device=dev)
    uu = uniform(seed, inst, st, OP_UT, m)
    us = torch.stack([0.5 * 9.81 * (1 + 0.1 * uu[..., 0]), 0.01 * uu[..., 1], 0.01 * uu[..., 2],
                      0.01 * uu[..., 3]], dim=-1)
    jac = torch.func.vmap(torch.func.jacrev(quadrotor_f, argnums=(0, 1)))
    Jx, Ju = jac(xs.reshape(-1, n), us.reshape(-1, m))
    eye = torch.eye(n, dtype=torch.float64, device=dev)
    A = colmajor(eye + dt * Jx).reshape(batch, N, n * n)
    B = colmajor(dt * Ju).reshape(batch, N, n * m)
    qd = torch.tensor([10, 10, 10, 1, 1, 1, 1, 1, 1, .1, .1, .1], dtype=torch.float64, device=dev)
    rd = torch.tensor([0.1, 1, 1, 1], dtype=torch.float64, device=dev)
    Q = pack_lower(torch.diag(qd)).expand(batch, N, sym_size(n)).contiguous()
    R = pack_lower(torch.diag(rd)).expand(batch, N, sym_size(m)).contiguous()
    xref = uniform(seed, inst, st, OP_XREF, n)
    q = -qd * xref
    xrefN = uniform(seed, inst, N, OP_XREF, n)
    return RRProblem(n, m, N, A=A.contiguous(), B=B.contiguous(), Q=Q,
                     M=torch.zeros(batch, N, n * m, dtype=torch.float64, device=dev), R=R, q=q.contiguous(),
                     r=torch.zeros(batch, N, m, dtype=torch.float64, device=dev),
                     c=(0.01 * uniform(seed, inst, st, OP_C, n)).contiguous(),
                     QN=pack_lower(torch.diag(10 * qd)).expand(batch, sym_size(n)).contiguous(),
                     qN=(-10 * qd * xrefN).contiguous(), c0=uniform(seed, inst, 0, OP_C0, n).contiguous(),
                     delta=torch.full((batch,), float(delta), dtype=torch.float64, device=dev))
