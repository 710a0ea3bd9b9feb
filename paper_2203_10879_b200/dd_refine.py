"""dd mode: the reference's own precision pair (hp = double-double, lp = binary64).

Mirrors `_run` (/root/reference/pkg/src/ddschur/refine.py:223-329) exactly as
the FP64-mode driver does, with
  hp products   Ozaki-II on the int8 tensor cores, beta = 102, double-double
                in and out (csrc/ozaki.cu, kind SR_MAT_DD) — replaces gemm_hp
                (_numba_kernels.py:18-46), whose dd EFT arithmetic costs ~184
                FP64 operations per complex MAC
  lp products   Ozaki-II, beta = 55, complex128 in and out (matmul_lp)
  lp solve      csrc/trisolve.cu in complex128 (solve_block, trisolve.py:243-262)
  Sigma         double-double sums left to right (orthogonal.py:191-200)
  row 0         the binary64 entry measurement (refine.py:126-135), as FP64
                Ozaki products of the hi parts
U = U_HP = 2^-106 in the stopping bound and the skip rule (refine.py:231,299-301).
"""
import math

import torch

from . import _lib, ozaki
from .errors import NormTooLarge, SeparationError
from .matmul import _counters, spectral_norm_estimate
from .matrix import DDPlanar, ZPlanar, lp_empty
from .trisolve import SolverWorkspace, solve_lp_device

U_HP = 2.0 ** -106
DIVERGENCE_STREAK = 3
_CLIP_HINT = ("clipping is disabled; retrying with clip_threshold=1e-5 may "
              "contain the blowup")


def _stream():
    return torch.cuda.current_stream().cuda_stream


class DDWorkspace:
    def __init__(self, n, device):
        self.n = n
        mk = lambda: DDPlanar.empty(n, device=device)  # noqa: E731
        self.q, self.q_next, self.p, self.that, self.y, self.sigma = mk(), mk(), mk(), mk(), mk(), mk()
        c128 = torch.complex128
        self.t_lp, self.e_lp, self.l_lp, self.w_lp, self.y_lp = (lp_empty(n, device=device, dtype=c128)
                                                                 for _ in range(5))
        self.yw, self.w2, self.w3 = (lp_empty(n, device=device, dtype=c128) for _ in range(3))
        self.w2y = self.w2yw = None
        self.q_c64 = lp_empty(n, device=device)
        self.scal = torch.zeros(8, dtype=torch.float64, device=device)
        red = _lib.load().sr_reduce_workspace_bytes()
        self.red = [torch.zeros(red, dtype=torch.uint8, device=device) for _ in range(6)]
        self.solver = SolverWorkspace(n, c128, device)
        self.row0 = ZPlanar.empty(n, device=device)  # binary64 scratch for the entry measurement

    def ptr(self, i):
        return self.scal.data_ptr() + 8 * i


class DDProducts:
    def __init__(self, ws, a):
        self.ws = ws
        n = ws.n
        dev = ws.q.hi.re_buf.device
        self.hp = ozaki.plan(n, ozaki.DD_BETA, ozaki.DD_BETA)
        self.lp = ozaki.plan(n, ozaki.DD_LP_BETA, ozaki.DD_LP_BETA)
        self.f64 = ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
        hp, lp = self.hp, self.lp
        self.ea_qh = ozaki.Encoded(n, n, 2, hp.beta_a, hp.nmod, dev)
        self.ea_x = ozaki.Encoded(n, n, 2, hp.beta_a, hp.nmod, dev)
        self.eb_q = ozaki.Encoded(n, n, 3, hp.beta_b, hp.nmod, dev)
        self.eb_s = ozaki.Encoded(n, n, 3, hp.beta_b, hp.nmod, dev)
        self.res = ozaki.ResidueBuffer(n, n, hp.nmod, dev)
        self.la = ozaki.Encoded(n, n, 2, lp.beta_a, lp.nmod, dev)
        self.lb = ozaki.Encoded(n, n, 3, lp.beta_b, lp.nmod, dev)
        self.lres = ozaki.ResidueBuffer(n, n, lp.nmod, dev)
        # a = None: products without A (the standalone newton_schulz_step /
        # merged_update of orthogonal.py)
        self.eb_a = ozaki.encode(a, n, n, "b", hp) if a is not None else None
        self.w_skew = True  # W exactly skew-Hermitian (W = L - L^H): W^2 / W^3 on the lower tiles
        self.a_hi = a.hi if a is not None else None

    def _hp(self, ea, eb, out, hermitian=False, **kw):
        ozaki.gemm_residues(ea, eb, self.hp, self.res, lower_only=hermitian)
        ozaki.decode(self.res, ea, eb, self.hp, out, hermitian=hermitian, **kw)
        _counters["hp_calls"] += 1

    def _lp(self, ea, eb, out, hermitian=False):
        ozaki.gemm_residues(ea, eb, self.lp, self.lres, lower_only=bool(hermitian))
        ozaki.decode(self.lres, ea, eb, self.lp, out, hermitian=hermitian)
        _counters["lp_calls"] += 1

    def entry(self, qhat):
        """Q = Q^ (3I - G) / 2 = Q^ - Q^ (G - I) / 2 in dd (orthogonal.py:167-169)."""
        ws, hp, n = self.ws, self.hp, self.ws.n
        ozaki.encode_dual(qhat, n, n, hp, self.ea_qh, self.eb_q)
        self._hp(self.ea_qh, self.eb_q, ws.y, shift=-1.0, hermitian=True)
        ozaki.encode(qhat, n, n, "a", hp, out=self.ea_x)
        ozaki.encode(ws.y, n, n, "b", hp, out=self.eb_s)
        self._hp(self.ea_x, self.eb_s, ws.q, alpha=-0.5, add=qhat)

    def entry_residuals(self, symmetric=False):
        """history row 0 (refine.py:126-135): (||stril(Q^H A Q)||, ||Q^H Q - I||)
        measured in binary64 on the hi parts of Q and A."""
        ws, n, f = self.ws, self.ws.n, self.f64
        q = ws.q.hi
        st = _stream()
        ea = ozaki.encode(q, n, n, "a", f, conj_t=True)
        eb_a = ozaki.encode(self.a_hi, n, n, "b", f)
        res = ozaki.ResidueBuffer(n, n, f.nmod, q.re_buf.device)
        ozaki.gemm_residues(ea, eb_a, f, res)
        ozaki.decode(res, ea, eb_a, f, ws.row0)                      # Q^H A
        ea_p = ozaki.encode(ws.row0, n, n, "a", f)
        eb_q = ozaki.encode(q, n, n, "b", f)
        ozaki.gemm_residues(ea_p, eb_q, f, res)
        ozaki.decode(res, ea_p, eb_q, f, ws.row0)                    # (Q^H A) Q
        t_lp = ws.t_lp
        _lib.call("sr_split_lp_c128", n, ws.row0.re_ptr(), ws.row0.im_ptr(), ws.row0.ld, t_lp.data_ptr(),
                  ws.e_lp.data_ptr(), t_lp.shape[1], ws.ptr(4), ws.red[4].data_ptr(), ws.red[4].numel(), st)
        if symmetric:  # + ||striu||: the full off-diagonal defect (refine.py:130-131)
            _lib.call("sr_striu_norm_f64", n, ws.row0.re_ptr(), ws.row0.im_ptr(), ws.row0.ld, ws.ptr(6),
                      ws.red[4].data_ptr(), ws.red[4].numel(), st)
        ozaki.gemm_residues(ea, eb_q, f, res, lower_only=True)
        ozaki.decode(res, ea, eb_q, f, ws.row0, shift=-1.0, hermitian=True)  # Q^H Q - I
        _lib.call("sr_fro_norm_f64", n, n, ws.row0.re_ptr(), ws.row0.im_ptr(), ws.row0.ld, ws.ptr(5),
                  ws.red[5].data_ptr(), ws.red[5].numel(), st)

    def measure(self):
        ws, hp, n = self.ws, self.hp, self.ws.n
        ozaki.encode_dual(ws.q, n, n, hp, self.ea_qh, self.eb_q)
        self._hp(self.ea_qh, self.eb_a, ws.p)
        ozaki.encode(ws.p, n, n, "a", hp, out=self.ea_x)
        self._hp(self.ea_x, self.eb_q, ws.that)
        self._hp(self.ea_qh, self.eb_q, ws.y, shift=-1.0, hermitian=True)

    def update(self, restore_full_sigma):
        ws, hp, lp, n = self.ws, self.hp, self.lp, self.ws.n
        st = _stream()
        _lib.call("sr_pack_c128", n, n, ws.y.hi.re_ptr(), ws.y.hi.im_ptr(), ws.y.ld, ws.y_lp.data_ptr(),
                  ws.y_lp.shape[1], st)
        ozaki.encode(ws.w_lp, n, n, "b", lp, out=self.lb)
        ozaki.encode(ws.y_lp, n, n, "a", lp, out=self.la)
        self._lp(self.la, self.lb, ws.yw)
        ozaki.encode(ws.w_lp, n, n, "a", lp, out=self.la)
        self._lp(self.la, self.lb, ws.w2, hermitian=self.w_skew)      # W skew-Hermitian: W^2 Hermitian
        ozaki.encode(ws.w2, n, n, "a", lp, out=self.la)
        self._lp(self.la, self.lb, ws.w3, hermitian="skew" if self.w_skew else False)  # W^3 skew-Hermitian
        w2y = w2yw = None
        if restore_full_sigma:
            if ws.w2y is None:
                ws.w2y = lp_empty(n, device=ws.w2.device, dtype=torch.complex128)
                ws.w2yw = lp_empty(n, device=ws.w2.device, dtype=torch.complex128)
            ozaki.encode(ws.y_lp, n, n, "b", lp, out=self.lb)
            ozaki.encode(ws.w2, n, n, "a", lp, out=self.la)
            self._lp(self.la, self.lb, ws.w2y)
            ozaki.encode(ws.w_lp, n, n, "b", lp, out=self.lb)
            ozaki.encode(ws.w2y, n, n, "a", lp, out=self.la)
            self._lp(self.la, self.lb, ws.w2yw)
            w2y, w2yw = ws.w2y.data_ptr(), ws.w2yw.data_ptr()
        y, s = ws.y, ws.sigma
        _lib.call("sr_sigma_merged_dd", n, ws.w_lp.data_ptr(), y.hi.re_ptr(), y.hi.im_ptr(), y.lo.re_ptr(),
                  y.lo.im_ptr(), y.ld, ws.yw.data_ptr(), ws.w2.data_ptr(), ws.w3.data_ptr(), w2y, w2yw,
                  ws.w_lp.shape[1], s.hi.re_ptr(), s.hi.im_ptr(), s.lo.re_ptr(), s.lo.im_ptr(), s.ld, 0, st)
        ozaki.encode(ws.q, n, n, "a", hp, out=self.ea_x)
        ozaki.encode(ws.sigma, n, n, "b", hp, out=self.eb_s)
        self._hp(self.ea_x, self.eb_s, ws.q_next, alpha=0.5, add=ws.q)
        ws.q, ws.q_next = ws.q_next, ws.q


_WS = {}


def _workspace(n, device):
    key = (n, str(device))
    if key not in _WS:
        _WS.clear()
        _WS[key] = DDWorkspace(n, device)
    return _WS[key]


def coerce_dd(x, device):
    """_coerce_hp (refine.py:341-350) for dd mode: DDPlanar, a 4-plane
    (re_hi, re_lo, im_hi, im_lo) tuple (DDMatrix.cells order) or any 2-d
    numpy / torch matrix (exact embedding, lo = 0)."""
    if isinstance(x, DDPlanar):
        m = x
    elif isinstance(x, ZPlanar):
        m = DDPlanar.from_any(x if not x.is_real else ZPlanar.from_any(x.re, device=device, force_complex=True),
                              device=device)
    else:
        m = DDPlanar.from_any(x, device=device)
    if m.rows != m.cols:
        raise ValueError("refinement needs a square matrix")
    from .refine import _finite_flag
    flags = torch.zeros(1, dtype=torch.int32, device=device)
    _finite_flag(m.hi, flags, 1)  # one libsr pass per pair of planes, one 4-byte read
    _finite_flag(m.lo, flags, 1)
    if int(flags.item()):
        raise ValueError("input matrix has non-finite entries")
    return m


def run_dd(a, qhat, cfg, device, symmetric=False):
    """_run in dd mode on DDPlanar inputs (symmetric: the Hermitian variant of
    refine_symmetric — full off-diagonal defect, diagonal-correction solve)."""
    from .refine import (RefineReport, RefineStatus, SchurPair, _exact_measure, _phase_permutation,
                         _quarter_phases, _structural_triangle)
    n = a.rows
    ws = _workspace(n, device)
    st = _stream()
    hp0 = _counters["hp_calls"]
    prod = DDProducts(ws, a)
    # entry Newton-Schulz guard (orthogonal.py:160-166), on the binary64 downcast
    _lib.call("sr_downcast_c64", n, n, qhat.hi.re_ptr(), qhat.hi.im_ptr(), qhat.ld, ws.q_c64.data_ptr(),
              ws.q_c64.shape[1], st)
    est = spectral_norm_estimate(ws.q_c64, n)
    if not est < math.sqrt(3.0):
        raise NormTooLarge("spectral norm estimate %.6f is not below sqrt(3)" % est)
    prod.entry(qhat)
    _lib.call("sr_fro_norm_f64", n, n, a.hi.re_ptr(), a.hi.im_ptr(), a.ld, ws.ptr(0), ws.red[0].data_ptr(),
              ws.red[0].numel(), st)
    prod.entry_residuals(symmetric)
    s = ws.scal.cpu()
    norm_a = float(s[0])
    history = [(math.hypot(float(s[4]), float(s[6])) if symmetric else float(s[4]), float(s[5]))]
    tol = cfg.tol_factor * n * U_HP * norm_a
    lo_zero = not (bool(ws.q.lo.re.any()) or bool(ws.q.lo.im.any()))
    perm = _phase_permutation(ws.q.hi) if lo_zero else None
    if perm is not None:
        t_exact = _structural_triangle(a.hi, ws.q.hi, perm, symmetric)
        if t_exact is not None:
            pair = SchurPair(q=ws.q, t=DDPlanar.from_any(t_exact, device=device), ortho_residual=history[0][1],
                             tri_residual=history[0][0])
            return pair, RefineReport(iterations=0, residual_history=history,
                                      hp_matmul_count=_counters["hp_calls"] - hp0, clipped_total=0,
                                      status=RefineStatus.CONVERGED, wall_time=0.0)
    status = RefineStatus.MAX_ITERS
    iterations = cfg.max_iters
    clipped_total = 0
    skip_fired = False
    detail = ""
    streak = 0
    ph = _quarter_phases(ws.q.hi, perm) if perm is not None else None
    for it in range(1, cfg.max_iters + 1):
        if ph is not None:  # Q a signed permutation: exact data movement (refine._exact_measure)
            _exact_measure(a, ph, perm, ws.that, ws.y)
        else:
            prod.measure()
        that = ws.that
        _lib.call("sr_split_lp_c128", n, that.hi.re_ptr(), that.hi.im_ptr(), that.ld, ws.t_lp.data_ptr(),
                  ws.e_lp.data_ptr(), ws.t_lp.shape[1], ws.ptr(1), ws.red[1].data_ptr(), ws.red[1].numel(), st)
        _lib.call("sr_fro_norm_f64", n, n, ws.y.hi.re_ptr(), ws.y.hi.im_ptr(), ws.y.ld, ws.ptr(2),
                  ws.red[2].data_ptr(), ws.red[2].numel(), st)
        if symmetric:
            _lib.call("sr_striu_norm_f64", n, that.hi.re_ptr(), that.hi.im_ptr(), that.ld, ws.ptr(6),
                      ws.red[1].data_ptr(), ws.red[1].numel(), st)
        s = ws.scal[:7].cpu()
        norm_e, norm_y = float(s[1]), float(s[2])
        if symmetric:
            norm_e = math.hypot(norm_e, float(s[6]))
        history.append((norm_e, norm_y))
        if not (math.isfinite(norm_e) and math.isfinite(norm_y)):
            status, iterations = RefineStatus.NON_FINITE, it
            detail = "iteration %d: residuals became non-finite" % it
            if cfg.clip_threshold is None:
                detail += "; " + _CLIP_HINT
            break
        converged = norm_e <= tol
        ws.solver.clipped.zero_()
        ws.solver.flags.zero_()
        if symmetric:
            clip = 0.0 if cfg.clip_threshold is None else float(cfg.clip_threshold)
            _lib.call("sr_diag_correction_c128", n, ws.t_lp.data_ptr(), ws.e_lp.data_ptr(), ws.t_lp.shape[1],
                      ws.l_lp.data_ptr(), clip, ws.solver.clipped.data_ptr(), ws.solver.flags.data_ptr(), st)
        else:
            solve_lp_device(ws.t_lp, ws.e_lp, ws.l_lp, n, cfg.clip_threshold, ws.solver, st)
        _lib.call("sr_skew_c128", n, ws.l_lp.data_ptr(), ws.l_lp.shape[1], ws.w_lp.data_ptr(), ws.ptr(3),
                  ws.solver.flags.data_ptr(), ws.red[3].data_ptr(), ws.red[3].numel(), st)
        norm_w = float(ws.scal[3].cpu())
        flags = int(ws.solver.flags.item())
        nclip = int(ws.solver.clipped.item())
        if flags & _lib.SR_FLAG_SEPARATION:
            raise SeparationError("repeated Ritz values: zero diagonal separation" if symmetric else
                                  "t has exactly repeated diagonal entries: diagonal separation is "
                                  "exactly zero")
        if flags & _lib.SR_FLAG_NONFINITE:
            status, iterations = RefineStatus.NON_FINITE, it
            detail = "iteration %d: %s" % (it, "diagonal correction solve overflowed" if symmetric else
                                           "solution contains non-finite entries")
            if cfg.clip_threshold is None:
                detail += "; " + _CLIP_HINT
            break
        clipped_total += nclip
        skip = (converged and cfg.skip_final_ortho and norm_y <= 10.0 * n * U_HP
                and norm_w <= math.sqrt(U_HP))
        if not skip:
            prod.update(cfg.restore_full_sigma)
            if ph is not None:  # still a signed permutation (W = 0: every correction clipped)?
                lo_zero = not (bool(ws.q.lo.re.any()) or bool(ws.q.lo.im.any()))
                perm = _phase_permutation(ws.q.hi) if lo_zero else None
                ph = _quarter_phases(ws.q.hi, perm)
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
    for z in (ws.that.hi, ws.that.lo):
        _lib.call("sr_triu_inplace_f64", n, z.re_ptr(), z.im_ptr(), z.ld, st)
        if symmetric:  # T keeps its real parts (refine.py:435-436)
            z.im.zero_()
    last_e, last_y = history[-1]
    q_out = DDPlanar(ZPlanar.empty(n, device=device), ZPlanar.empty(n, device=device))
    t_out = DDPlanar(ZPlanar.empty(n, device=device), ZPlanar.empty(n, device=device))
    for dst, src in ((q_out.hi, ws.q.hi), (q_out.lo, ws.q.lo), (t_out.hi, ws.that.hi), (t_out.lo, ws.that.lo)):
        dst.copy_(src)
    pair = SchurPair(q=q_out, t=t_out, ortho_residual=last_y, tri_residual=last_e)
    report = RefineReport(iterations=iterations, residual_history=history,
                          hp_matmul_count=_counters["hp_calls"] - hp0, clipped_total=clipped_total,
                          status=status, wall_time=0.0, skip_fired=skip_fired, detail=detail)
    return pair, report
