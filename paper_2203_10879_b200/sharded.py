"""Multi-GPU refinement: products sharded by output columns over P ranks.

Same loop as refine._run_fp64 (itself `_run`, /root/reference/pkg/src/ddschur/
refine.py:223-329).  Rank r owns the column block J_r of T^, Y, S' and Q_new;
A, the current Q (FP64) and the lp matrices of the solve are replicated.
Per iteration, with the single-GPU product set (Gaussian-CRT planes, DESIGN.md
§3.0) restricted to the block:

  measure  Q encoded once as a B operand (Gaussian planes; read with swapped
           planes it is the A operand of Q^H, ozaki.conj_view);
           Y_J = Q^H Q_J - I_J, Z_J = A Q_J (A encoded once per refinement,
           real A as one plane pair), T^_J = Q^H Z_J;
           split + lp downcast of the block, partial squared norms
           -> one all-reduce of two scalars, all-gathers of lp T, E (the
           replicated solve's input)
  solve    replicated (deterministic: every rank holds the identical W)
  update   W^2_J = W W_J and X W_J with X = Y - W - W^2 (the fused two-product
           form, magnitude-adaptive lp plans, products.lp_plans), one all-gather
           of the lp X blocks; S'_J; Q_new_J = Q_J + Q S'_J / 2 at the
           correction plan (ozaki.correction_beta); one all-gather of Q_new.

Per rank and iteration: (3 hp + 2 lp products) / P, the full-Q encodes
(one B-role hq encoding, one A-role encoding at the shrinking correction
plan), the replicated solve, and all-gathers of 2 lp + 1 lp + 1 FP64 matrices
(~2.5 GB received at n = 8192).  DESIGN.md §6 has the per-P model; the solve
is the Amdahl term.

The driver is written against a small backend protocol so its control flow
(sharding, gathers, reductions, statuses) is exercised by world-size-2 gloo
tests on the CPU (tests/test_parallel.py) with a reference-arithmetic
backend; `OzakiShardBackend` is the GPU implementation on libsr.
"""
import math

import torch
import torch.distributed as dist

from . import _lib, ozaki, parallel, products
from .errors import NormTooLarge, SeparationError
from .matmul import _counters, spectral_norm_estimate
from .matrix import ColView, ZPlanar, lp_empty
from .trisolve import SolverWorkspace, solve_lp_device

U_FP64 = 2.0 ** -53
DIVERGENCE_STREAK = 3


def refine_sharded(backend, cfg, group=None, align=128):
    """Run the FP64-mode refinement on `backend` (already holding A and Q^);
    returns (q_full, t_full, report fields dict) identical on every rank.
    hp_matmul_count is the reference's logical count (refine.py:7-10), not
    the per-rank launches."""
    from .refine import RefineStatus
    rank, world = parallel.world_info(group)
    n = backend.n
    ranges = parallel.column_ranges(n, world, align)
    j0, j1 = ranges[rank]
    be = backend
    be.set_columns(j0, j1, ranges, group)
    hp = 0
    be.norm_guard()
    be.entry_cols()
    hp += 2
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
        hp += 3
        norm_e, norm_y = be.norms()
        if it == 1:
            history.append((norm_e, norm_y))
        history.append((norm_e, norm_y))
        if not (math.isfinite(norm_e) and math.isfinite(norm_y)):
            status, iterations = RefineStatus.NON_FINITE, it
            detail = "iteration %d: residuals became non-finite" % it
            break
        converged = norm_e <= tol
        be.gather_lp()
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
            be.update_cols(norm_y, norm_w)
            hp += 1
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
    _counters["hp_calls"] += hp
    return q, t, dict(iterations=iterations, residual_history=history, hp_matmul_count=hp,
                      clipped_total=clipped_total, status=status, skip_fired=skip_fired, detail=detail)


def _stream():
    return torch.cuda.current_stream().cuda_stream


class OzakiShardBackend:
    """Column-sharded FP64-mode products on the int8 tensor cores (libsr),
    Gaussian-CRT planes (two real products per modulus, ozaki.py)."""

    def __init__(self, a, qhat, device):
        self.dev = device
        self.a = ZPlanar.from_any(a, device=device)
        self.qhat = ZPlanar.from_any(qhat, device=device, force_complex=True)
        n = self.n = self.a.rows
        self.q = ZPlanar.empty(n, device=device)
        self.t_lp, self.e_lp, self.l_lp, self.w_lp, self.y_lp, self.x_lp = (lp_empty(n, device=device)
                                                                            for _ in range(6))
        self.scal = torch.zeros(8, dtype=torch.float64, device=device)
        red = _lib.load().sr_reduce_workspace_bytes()
        self.red = [torch.zeros(red, dtype=torch.uint8, device=device) for _ in range(4)]
        self.solver = SolverWorkspace(n, torch.complex64, device)
        bq = ozaki.HP_BETA_Q
        self.hq = ozaki.gauss_plan(n, bq, bq)                  # Q^H Q_J (and G - I at the entry)
        self.hp_z = ozaki.gauss_plan(n, ozaki.HP_BETA, bq)     # Z_J = A Q_J
        self.hp_t = ozaki.gauss_plan(n, bq, ozaki.HP_BETA)     # T^_J = Q^H Z_J
        self.lp = ozaki.gauss_plan(n, ozaki.LP_BETA, ozaki.LP_BETA)
        self.ea_a = None  # A, A role: encoded at the first measurement, kept for the refinement

    # ---- sharding
    def set_columns(self, j0, j1, ranges, group):
        n, dev = self.n, self.dev
        self.j0, self.j1, self.ranges, self.group = j0, j1, ranges, group
        w = self.w = j1 - j0  # >= 1 (parallel.column_ranges)
        self.zj, self.tj, self.yj, self.sj, self.qj = (ZPlanar.empty(n, w, device=dev) for _ in range(5))
        self.wj, self.w2j, self.xwj, self.xj, self.t_lpj, self.e_lpj, self.y_lpj = (lp_empty(n, w, device=dev)
                                                                                   for _ in range(7))
        nm, lm = self.hq.nmod, self.lp.nmod
        self.eq = ozaki.Encoded(n, n, 2, ozaki.HP_BETA_Q, nm, dev)   # full Q, B role (+ Q^H read swapped)
        self.eb_j = ozaki.Encoded(w, n, 2, ozaki.HP_BETA, nm, dev)   # B operand blocks: Q_J, Z_J, S'_J, (G - I)_J
        self.ea_x = ozaki.Encoded(n, n, 2, ozaki.HP_BETA, nm, dev)   # Q^ / Q, A role, correction plans
        self.res = ozaki.ResidueBuffer(n, w, nm, dev)
        self.la = ozaki.Encoded(n, n, 2, ozaki.LP_BETA, lm, dev)     # W / X, A role
        self.lb = ozaki.Encoded(w, n, 2, ozaki.LP_BETA, lm, dev)     # W_J, B role
        self.lres = ozaki.ResidueBuffer(n, w, lm, dev)
        self.gather = parallel.ColGatherer(ranges, group)

    def _cols(self, z):
        return ColView(z, self.j0, self.j1)

    def _prod(self, pl, ea, eb, res, out, **kw):
        ozaki.gemm_residues(ea, eb, pl, res)
        ozaki.decode(res, ea, eb, pl, out, **kw)

    def _gather_planar(self, local, full):
        self.gather(local.re, full.re_buf)
        self.gather(local.im, full.im_buf)

    def _gather_lp(self, local, full):
        n, w = self.n, self.w
        self.gather(torch.view_as_real(local[:, :w]), torch.view_as_real(full[:, :n]))

    def _all_reduce(self, t):
        if parallel.world_info(self.group)[1] > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def _block_sq_norm(self, z, slot):
        """||z_J||_F^2 of a planar n x w block into scal[slot] (squared on the device)."""
        _lib.call("sr_fro_norm_f64", self.n, self.w, z.re_ptr(), z.im_ptr(), z.ld, self.scal.data_ptr() + 8 * slot,
                  self.red[slot % 4].data_ptr(), self.red[slot % 4].numel(), _stream())
        self.scal[slot:slot + 1].square_()

    # ---- steps
    def norm_guard(self):
        n = self.n
        _lib.call("sr_downcast_c64", n, n, self.qhat.re_ptr(), self.qhat.im_ptr(), self.qhat.ld,
                  self.y_lp.data_ptr(), self.y_lp.shape[1], _stream())
        est = spectral_norm_estimate(self.y_lp, n)
        if not est < math.sqrt(3.0):
            raise NormTooLarge("spectral norm estimate %.6f is not below sqrt(3)" % est)

    def entry_cols(self):
        """Q[:, J] = Q^[:, J] - Q^ (Q^H Q^[:, J] - I_J) / 2 (orthogonal.py:167-169)."""
        n, w, hq = self.n, self.w, self.hq
        ozaki.encode(self.qhat, n, n, "b", hq, out=self.eq)
        ozaki.encode(self._cols(self.qhat), n, w, "b", hq, out=self.eb_j)
        self._prod(hq, ozaki.conj_view(self.eq), self.eb_j, self.res, self.yj, shift=-1.0, diag_col0=self.j0)
        self._block_sq_norm(self.yj, 4)
        bound = math.sqrt(float(self._all_reduce(self.scal[4:5].clone()).item()))
        pc = ozaki.correction_plan(bound, n)
        ozaki.encode(self.qhat, n, n, "a", pc, out=self.ea_x)
        ozaki.encode(self.yj, n, w, "b", pc, out=self.eb_j)
        self._prod(pc, self.ea_x, self.eb_j, self.res, self.qj, alpha=-0.5, add=self._cols(self.qhat))

    def gather_q(self):
        self._gather_planar(self.qj, self.q)

    def norm_a(self):
        n = self.n
        _lib.call("sr_fro_norm_f64", n, n, self.a.re_ptr(), self.a.im_ptr(), self.a.ld, self.scal.data_ptr(),
                  self.red[0].data_ptr(), self.red[0].numel(), _stream())
        return float(self.scal[0].cpu())

    def measure_cols(self):
        """Y_J = Q^H Q_J - I_J, Z_J = A Q_J, T^_J = Q^H Z_J; split + partial norms."""
        n, w, j0, st = self.n, self.w, self.j0, _stream()
        ozaki.encode(self.q, n, n, "b", self.hq, out=self.eq)      # Q (B role); Q^H = its swapped planes
        qh = ozaki.conj_view(self.eq)
        if self.ea_a is None:
            self.ea_a = ozaki.encode(self.a, n, n, "a", self.hp_z)
        ozaki.encode(self._cols(self.q), n, w, "b", self.hq, out=self.eb_j)
        self._prod(self.hq, qh, self.eb_j, self.res, self.yj, shift=-1.0, diag_col0=j0)
        self._prod(self.hp_z, self.ea_a, self.eb_j, self.res, self.zj)
        ozaki.encode(self.zj, n, w, "b", self.hp_t, out=self.eb_j)
        self._prod(self.hp_t, qh, self.eb_j, self.res, self.tj)
        _lib.call("sr_split_lp_block_c64", n, w, j0, self.tj.re_ptr(), self.tj.im_ptr(), self.tj.ld,
                  self.t_lpj.data_ptr(), self.e_lpj.data_ptr(), self.t_lpj.shape[1], self.scal.data_ptr() + 8,
                  self.red[1].data_ptr(), self.red[1].numel(), st)
        self._block_sq_norm(self.yj, 2)
        _lib.call("sr_downcast_c64", n, w, self.yj.re_ptr(), self.yj.im_ptr(), self.yj.ld, self.y_lpj.data_ptr(),
                  self.y_lpj.shape[1], st)

    def norms(self):
        s = self._all_reduce(self.scal[1:3].clone()).cpu()
        return math.sqrt(float(s[0])), math.sqrt(float(s[1]))

    def gather_lp(self):
        self._gather_lp(self.t_lpj, self.t_lp)
        self._gather_lp(self.e_lpj, self.e_lp)

    def solve(self, clip):
        n, st = self.n, _stream()
        self.solver.clipped.zero_()
        self.solver.flags.zero_()
        solve_lp_device(self.t_lp, self.e_lp, self.l_lp, n, clip, self.solver, st)
        _lib.call("sr_skew_c64", n, self.l_lp.data_ptr(), self.l_lp.shape[1], self.w_lp.data_ptr(),
                  self.scal.data_ptr() + 24, self.solver.flags.data_ptr(), self.red[3].data_ptr(),
                  self.red[3].numel(), st)
        return float(self.scal[3].cpu()), int(self.solver.flags.item()), int(self.solver.clipped.item())

    def update_cols(self, norm_y, norm_w):
        """W^2_J, X_J = Y_J - W_J - W^2_J (gathered), (X W)_J, S'_J,
        Q_new_J = Q_J + Q S'_J / 2 (orthogonal.py:172-201, fused form)."""
        n, w, j0, j1, st = self.n, self.w, self.j0, self.j1, _stream()
        p_w2, p_xw = products.lp_plans(n, norm_y, norm_w, True, self.lp)
        # lp products below their own error budget are not formed (products.lp_skips;
        # the norms are all-reduced, so every rank decides alike)
        skip_w2, skip_xw = products.lp_skips(norm_y, norm_w)
        self.wj[:, :w].copy_(self.w_lp[:, j0:j1])
        xw = None
        if not skip_xw:
            w_plan = None
            if not skip_w2:
                ozaki.encode(self.w_lp, n, n, "a", p_w2, out=self.la)     # W (replicated), A role
                ozaki.encode(self.wj, n, w, "b", p_w2, out=self.lb)       # W_J, B role
                self._prod(p_w2, self.la, self.lb, self.lres, self.w2j)   # W^2_J
                w_plan = p_w2
            _lib.call("sr_fused_lp_operand_block_c64", n, w, self.yj.re_ptr(), self.yj.im_ptr(), self.yj.ld,
                      self.wj.data_ptr(), None if skip_w2 else self.w2j.data_ptr(), self.wj.shape[1],
                      self.xj.data_ptr(), st)
            self._gather_lp(self.xj, self.x_lp)                      # X = Y - W - W^2 (full)
            if p_xw is not w_plan:
                ozaki.encode(self.wj, n, w, "b", p_xw, out=self.lb)
            ozaki.encode(self.x_lp, n, n, "a", p_xw, out=self.la)
            self._prod(p_xw, self.la, self.lb, self.lres, self.xwj)   # (X W)_J = (YW - W^2 - W^3)_J
            xw = self.xwj.data_ptr()
        _lib.call("sr_sigma_merged_f64", n, w, self.wj.data_ptr(), self.yj.re_ptr(), self.yj.im_ptr(), self.yj.ld,
                  xw, None, None, None, None, self.wj.shape[1], self.sj.re_ptr(), self.sj.im_ptr(),
                  self.sj.ld, 0, st)                                  # S'_J = 2 W_J - Y_J - (X W)_J
        bound = products.sigma_prime_bound(norm_y, norm_w, False)
        pc = ozaki.correction_plan(bound, n)
        ozaki.encode(self.q, n, n, "a", pc, out=self.ea_x)
        ozaki.encode(self.sj, n, w, "b", pc, out=self.eb_j)
        self._prod(pc, self.ea_x, self.eb_j, self.res, self.qj, alpha=0.5, add=self._cols(self.q))

    def result(self):
        n, st = self.n, _stream()
        that = ZPlanar.empty(n, device=self.dev)
        self._gather_planar(self.tj, that)
        _lib.call("sr_triu_inplace_f64", n, that.re_ptr(), that.im_ptr(), that.ld, st)
        return self.q.to_complex(), that.to_complex()


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
