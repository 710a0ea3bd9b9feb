"""Multi-GPU refinement: products sharded by output columns over P ranks.

Same loop as refine._run_fp64 (itself `_run`, /root/reference/pkg/src/ddschur/
refine.py:223-329); every hp / lp product is split by output columns
(parallel.py), the solver runs replicated on the gathered lp T^ (so every
rank holds the identical correction W and no broadcast is needed), and the
status logic sees identical scalars on every rank.  Per iteration each rank
computes 1/P of all products and receives (P-1)/P of T^ and Y (hp), W^2 (lp)
and Q_new (hp) — about 3.5 GB at n = 8192 — over NVLink.

The driver is written against a small backend protocol so its control flow
(sharding, gathers, reductions, statuses) is exercised by world-size-2 gloo
tests on the CPU (tests/test_parallel.py) with a reference-arithmetic
backend; `OzakiShardBackend` is the GPU implementation on libsr.
"""
import math

import torch

from . import _lib, ozaki, parallel
from .errors import NormTooLarge, SeparationError
from .matmul import _counters, spectral_norm_estimate
from .matrix import ColView, ZPlanar, lp_empty
from .trisolve import SolverWorkspace, solve_lp_device

U_FP64 = 2.0 ** -53
DIVERGENCE_STREAK = 3


def refine_sharded(backend, cfg, group=None, align=128):
    """Run the FP64-mode refinement on `backend` (already holding A and Q^);
    returns (q_full, t_full, report fields dict) identical on every rank."""
    from .refine import RefineStatus
    rank, world = parallel.world_info(group)
    n = backend.n
    ranges = parallel.column_ranges(n, world, align)
    j0, j1 = ranges[rank]
    be = backend
    be.set_columns(j0, j1, ranges, group)
    hp0 = _counters["hp_calls"]
    be.norm_guard()
    be.entry_cols()
    be.gather_q()
    norm_a = be.norm_a()
    tol = cfg.tol_factor * n * U_FP64 * norm_a
    history = []
    status = RefineStatus.MAX_ITERS
    iterations = cfg.max_iters
    clipped_total = 0
    skip_fired = False
    detail = ""
    streak = 0
    for it in range(1, cfg.max_iters + 1):
        be.measure_cols()
        be.gather_that_y()
        norm_e, norm_y = be.norms()
        if it == 1:
            history.append((norm_e, norm_y))
        history.append((norm_e, norm_y))
        if not (math.isfinite(norm_e) and math.isfinite(norm_y)):
            status, iterations = RefineStatus.NON_FINITE, it
            detail = "iteration %d: residuals became non-finite" % it
            break
        converged = norm_e <= tol
        norm_w, flags, nclip = be.solve(cfg.clip_threshold)
        if flags & _lib.SR_FLAG_SEPARATION:
            raise SeparationError("t has exactly repeated diagonal entries: diagonal separation is exactly zero")
        if flags & _lib.SR_FLAG_NONFINITE:
            status, iterations = RefineStatus.NON_FINITE, it
            detail = "iteration %d: solution contains non-finite entries" % it
            break
        clipped_total += nclip
        skip = (converged and cfg.skip_final_ortho and norm_y <= 10.0 * n * U_FP64
                and norm_w <= math.sqrt(U_FP64))
        if not skip:
            be.update_stage1_cols()
            be.gather_w2()
            be.update_stage2_cols()
            be.gather_q()
        if converged:
            status, iterations, skip_fired = RefineStatus.CONVERGED, it, skip
            break
        if len(history) >= 2 and norm_e > history[-2][0]:
            streak += 1
        else:
            streak = 0
        if streak >= DIVERGENCE_STREAK:
            status, iterations = RefineStatus.DIVERGED, it
            break
    q, t = be.result()
    return q, t, dict(iterations=iterations, residual_history=history,
                      hp_matmul_count=_counters["hp_calls"] - hp0, clipped_total=clipped_total,
                      status=status, skip_fired=skip_fired, detail=detail)


class OzakiShardBackend:
    """Column-sharded FP64-mode products on the int8 tensor cores (libsr),
    Gaussian-CRT planes (two real products per modulus, ozaki.py)."""

    def __init__(self, a, qhat, device):
        self.dev = device
        self.a = ZPlanar.from_any(a, device=device)
        self.qhat = ZPlanar.from_any(qhat, device=device, force_complex=True)
        n = self.n = self.a.rows
        self.q = ZPlanar.empty(n, device=device)
        self.that = ZPlanar.empty(n, device=device)
        self.y = ZPlanar.empty(n, device=device)
        self.t_lp, self.e_lp, self.l_lp, self.w_lp, self.y_lp, self.w2 = (lp_empty(n, device=device)
                                                                           for _ in range(6))
        self.scal = torch.zeros(8, dtype=torch.float64, device=device)
        red = _lib.load().sr_reduce_workspace_bytes()
        self.red = [torch.zeros(red, dtype=torch.uint8, device=device) for _ in range(4)]
        self.solver = SolverWorkspace(n, torch.complex64, device)
        self.hp = ozaki.gauss_plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
        self.lp = ozaki.gauss_plan(n, ozaki.LP_BETA, ozaki.LP_BETA)
        self.ea_a = ozaki.encode(self.a, n, n, "a", self.hp)  # A, A role (Z_J = A Q_J)

    # ---- sharding
    def set_columns(self, j0, j1, ranges, group):
        n, dev, hp, lp = self.n, self.dev, self.hp, self.lp
        self.j0, self.j1, self.ranges, self.group = j0, j1, ranges, group
        w = self.w = max(j1 - j0, 1)
        self.zj, self.tj, self.yj, self.sj, self.qj = (ZPlanar.empty(n, w, device=dev) for _ in range(5))
        self.ywj, self.w2j, self.w3j, self.wj = (lp_empty(n, w, device=dev) for _ in range(4))
        self.ea_full = ozaki.Encoded(n, n, 2, hp.beta_a, hp.nmod, dev)
        self.eb_cols = ozaki.Encoded(w, n, 2, hp.beta_b, hp.nmod, dev)
        self.res = ozaki.ResidueBuffer(n, w, hp.nmod, dev)
        self.la = ozaki.Encoded(n, n, 2, lp.beta_a, lp.nmod, dev)
        self.lb = ozaki.Encoded(w, n, 2, lp.beta_b, lp.nmod, dev)
        self.lres = ozaki.ResidueBuffer(n, w, lp.nmod, dev)

    def _cols(self, z):
        return ColView(z, self.j0, self.j1)

    def _hp(self, ea, eb, out, **kw):
        ozaki.gemm_residues(ea, eb, self.hp, self.res)
        ozaki.decode(self.res, ea, eb, self.hp, out, **kw)

    def _lp(self, ea, eb, out):
        ozaki.gemm_residues(ea, eb, self.lp, self.lres)
        ozaki.decode(self.lres, ea, eb, self.lp, out)

    def _gather_planar(self, local, full):
        parallel.all_gather_cols(local.re, full.re, self.ranges, self.group)
        parallel.all_gather_cols(local.im, full.im, self.ranges, self.group)

    def _gather_lp(self, local, full):
        n, w = self.n, self.j1 - self.j0
        parallel.all_gather_cols(torch.view_as_real(local[:, :w]), torch.view_as_real(full[:, :n]), self.ranges,
                                 self.group)

    # ---- steps
    def norm_guard(self):
        n = self.n
        q_lp = self.y_lp
        _lib.call("sr_downcast_c64", n, n, self.qhat.re_ptr(), self.qhat.im_ptr(), self.qhat.ld, q_lp.data_ptr(),
                  q_lp.shape[1], torch.cuda.current_stream().cuda_stream)
        est = spectral_norm_estimate(q_lp, n)
        if not est < math.sqrt(3.0):
            raise NormTooLarge("spectral norm estimate %.6f is not below sqrt(3)" % est)

    def entry_cols(self):
        """Q[:, J] = Q^[:, J] - Q^ (Q^H Q^[:, J] - I_J) / 2."""
        n, hp, w = self.n, self.hp, self.j1 - self.j0
        ozaki.encode(self.qhat, n, n, "a", hp, conj_t=True, out=self.ea_full)
        ozaki.encode(self._cols(self.qhat), n, w, "b", hp, out=self.eb_cols)
        self._hp(self.ea_full, self.eb_cols, self.yj, shift=-1.0, diag_col0=self.j0)
        ozaki.encode(self.qhat, n, n, "a", hp, out=self.ea_full)
        ozaki.encode(self.yj, n, w, "b", hp, out=self.eb_cols)
        self._hp(self.ea_full, self.eb_cols, self.qj, alpha=-0.5, add=self._cols(self.qhat))
        _counters["hp_calls"] += 2

    def gather_q(self):
        self._gather_planar(self.qj, self.q)

    def norm_a(self):
        n = self.n
        _lib.call("sr_fro_norm_f64", n, n, self.a.re_ptr(), self.a.im_ptr(), self.a.ld, self.scal.data_ptr(),
                  self.red[0].data_ptr(), self.red[0].numel(), torch.cuda.current_stream().cuda_stream)
        return float(self.scal[0].cpu())

    def measure_cols(self):
        """T^[:, J] = Q^H (A Q[:, J]), Y[:, J] = Q^H Q[:, J] - I_J."""
        n, hp, w = self.n, self.hp, self.j1 - self.j0
        ozaki.encode(self._cols(self.q), n, w, "b", hp, out=self.eb_cols)
        self._hp(self.ea_a, self.eb_cols, self.zj)                                   # Z_J = A Q_J
        ozaki.encode(self.q, n, n, "a", hp, conj_t=True, out=self.ea_full)
        self._hp(self.ea_full, self.eb_cols, self.yj, shift=-1.0, diag_col0=self.j0)  # Y_J
        ozaki.encode(self.zj, n, w, "b", hp, out=self.eb_cols)
        self._hp(self.ea_full, self.eb_cols, self.tj)                                # T^_J
        _counters["hp_calls"] += 3

    def gather_that_y(self):
        self._gather_planar(self.tj, self.that)
        self._gather_planar(self.yj, self.y)

    def norms(self):
        n, st = self.n, torch.cuda.current_stream().cuda_stream
        _lib.call("sr_split_lp_c64", n, self.that.re_ptr(), self.that.im_ptr(), self.that.ld, self.t_lp.data_ptr(),
                  self.e_lp.data_ptr(), self.t_lp.shape[1], self.scal.data_ptr() + 8, self.red[1].data_ptr(),
                  self.red[1].numel(), st)
        _lib.call("sr_fro_norm_f64", n, n, self.y.re_ptr(), self.y.im_ptr(), self.y.ld, self.scal.data_ptr() + 16,
                  self.red[2].data_ptr(), self.red[2].numel(), st)
        s = self.scal[1:3].cpu()
        return float(s[0]), float(s[1])

    def solve(self, clip):
        n, st = self.n, torch.cuda.current_stream().cuda_stream
        self.solver.clipped.zero_()
        self.solver.flags.zero_()
        solve_lp_device(self.t_lp, self.e_lp, self.l_lp, n, clip, self.solver, st)
        _lib.call("sr_skew_c64", n, self.l_lp.data_ptr(), self.l_lp.shape[1], self.w_lp.data_ptr(),
                  self.scal.data_ptr() + 24, self.solver.flags.data_ptr(), self.red[3].data_ptr(),
                  self.red[3].numel(), st)
        return float(self.scal[3].cpu()), int(self.solver.flags.item()), int(self.solver.clipped.item())

    def update_stage1_cols(self):
        """Y W[:, J] and W W[:, J] (lp)."""
        n, lp, w = self.n, self.lp, self.j1 - self.j0
        st = torch.cuda.current_stream().cuda_stream
        _lib.call("sr_downcast_c64", n, n, self.y.re_ptr(), self.y.im_ptr(), self.y.ld, self.y_lp.data_ptr(),
                  self.y_lp.shape[1], st)
        self.wj[:, :w].copy_(self.w_lp[:, self.j0:self.j1])
        ozaki.encode(self.wj, n, w, "b", lp, out=self.lb)
        ozaki.encode(self.y_lp, n, n, "a", lp, out=self.la)
        self._lp(self.la, self.lb, self.ywj)
        ozaki.encode(self.w_lp, n, n, "a", lp, out=self.la)
        self._lp(self.la, self.lb, self.w2j)

    def gather_w2(self):
        self._gather_lp(self.w2j, self.w2)

    def update_stage2_cols(self):
        """W^3[:, J], Sigma'[:, J], Q_new[:, J] = Q_J + Q Sigma'_J / 2."""
        n, lp, hp, w = self.n, self.lp, self.hp, self.j1 - self.j0
        st = torch.cuda.current_stream().cuda_stream
        ozaki.encode(self.w2, n, n, "a", lp, out=self.la)
        self._lp(self.la, self.lb, self.w3j)
        # Sigma'_J (n x w block; the lp blocks share ywj's leading dimension)
        _lib.call("sr_sigma_merged_f64", n, w, self.wj.data_ptr(), self.yj.re_ptr(), self.yj.im_ptr(), self.yj.ld,
                  self.ywj.data_ptr(), self.w2j.data_ptr(), self.w3j.data_ptr(), None, None, self.wj.shape[1],
                  self.sj.re_ptr(), self.sj.im_ptr(), self.sj.ld, 0, st)
        ozaki.encode(self.q, n, n, "a", hp, out=self.ea_full)
        ozaki.encode(self.sj, n, w, "b", hp, out=self.eb_cols)
        self._hp(self.ea_full, self.eb_cols, self.qj, alpha=0.5, add=self._cols(self.q))
        _counters["hp_calls"] += 1

    def result(self):
        n, st = self.n, torch.cuda.current_stream().cuda_stream
        _lib.call("sr_triu_inplace_f64", n, self.that.re_ptr(), self.that.im_ptr(), self.that.ld, st)
        return self.q.to_complex(), self.that.to_complex()


def refine_template_distributed(a, qhat, cfg=None, group=None, device=None):
    """refine_template (refine.py:357-380) on every rank of `group`, products
    sharded by columns; returns the same (SchurPair, RefineReport) on every
    rank.  FP64 mode only."""
    import time

    from .refine import RefineConfig, RefineReport, SchurPair
    cfg = RefineConfig(precision="fp64") if cfg is None else cfg
    if cfg.precision != "fp64":
        raise NotImplementedError("the sharded driver runs FP64 mode")
    device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    t0 = time.perf_counter()
    be = OzakiShardBackend(a, qhat, device)
    q, t, rep = refine_sharded(be, cfg, group)
    torch.cuda.current_stream().synchronize()
    last_e, last_y = rep["residual_history"][-1]
    pair = SchurPair(q=q, t=t, ortho_residual=last_y, tri_residual=last_e)
    return pair, RefineReport(wall_time=time.perf_counter() - t0, **rep)
