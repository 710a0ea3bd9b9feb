"""Newton-like Schur refinement on the B200: the drop-in `refine_template`.

Mirrors the reference driver and loop
  RefineConfig / RefineReport / RefineStatus  /root/reference/pkg/src/ddschur/refine.py:39-102
  refine_template                             refine.py:357-380
  _run (the loop)                             refine.py:223-329
  _finish / _coerce_hp                        refine.py:332-350
  newton_schulz_step / merged_update          orthogonal.py:153-201
with every matrix operation in libsr.so.  One extra config field,
`precision`, selects the precision pair:
  "fp64": hp = FP64 complex (DMMA GEMMs), lp = complex64 (the BASELINE
          configs 1, 2, 3, 5; U = 2^-53 in the stopping bound and skip rule);
  "dd":   hp = double-double, lp = binary64 — the reference's own pair.
The host loop reads back two small scalar groups per iteration (the norms
after T^/Y, then ||W|| + flags + clip count after the solve); everything
else stays on the device.
"""
import dataclasses
import enum
import math
import time

from typing import NamedTuple

import numpy as np
import torch

from . import _lib, products
from .errors import NonFiniteError, NormTooLarge, NotSymmetric, SeparationError  # noqa: F401
from .matmul import _counters, matmul_hp, spectral_norm_estimate
from .matrix import ZPlanar, lp_empty
from .trisolve import SolverWorkspace, solve_lp_device

U_HP = 2.0 ** -106
U_FP64 = 2.0 ** -53

DIVERGENCE_STREAK = 3
_CLIP_HINT = ("clipping is disabled; retrying with clip_threshold=1e-5 may "
              "contain the blowup")


class OrthoStrategy(enum.Enum):
    QR_RETRACTION = "qr"
    NEWTON_SCHULZ = "ns"


class RefineStatus(enum.Enum):
    CONVERGED = "Converged"
    MAX_ITERS = "MaxIters"
    DIVERGED = "Diverged"
    NON_FINITE = "NonFinite"


@dataclasses.dataclass
class RefineConfig:
    """refine.py:53-82, plus `precision` ("fp64" | "dd") and `gemm`
    ("ozaki": int8 tensor-core Ozaki-II products on Gaussian-CRT planes,
    default; "ozaki_std": the same with (re, im) planes, four real products
    per complex one; "dmma": FP64 DMMA / FP32 SIMT products)."""

    tol_factor: float = 10.0
    max_iters: int = 20
    n_min: int = 4
    clip_threshold: float | None = None
    ortho: OrthoStrategy = OrthoStrategy.NEWTON_SCHULZ
    skip_final_ortho: bool = True
    seed: int = 0
    restore_full_sigma: bool = False
    precision: str = "dd"
    gemm: str = "ozaki"

    def __post_init__(self):
        if not self.tol_factor > 0.0:
            raise ValueError("tol_factor must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be at least 1")
        if self.n_min < 2:
            raise ValueError("n_min must be at least 2")
        if self.clip_threshold is not None and not self.clip_threshold > 0.0:
            raise ValueError("clip_threshold must be positive when set")
        if not isinstance(self.ortho, OrthoStrategy):
            raise ValueError("ortho must be an OrthoStrategy")
        if self.precision not in ("fp64", "dd"):
            raise ValueError("precision must be 'fp64' or 'dd'")
        if self.gemm not in ("ozaki", "ozaki_std", "dmma"):
            raise ValueError("gemm must be 'ozaki', 'ozaki_std' or 'dmma'")


@dataclasses.dataclass
class RefineReport:
    """refine.py:85-102."""

    iterations: int
    residual_history: list
    hp_matmul_count: int
    clipped_total: int
    status: RefineStatus
    wall_time: float
    skip_fired: bool = False
    detail: str = ""


@dataclasses.dataclass
class SchurPair:
    """schur.py:29-49: q unitary, t upper triangular (device tensors)."""

    q: object
    t: object
    ortho_residual: float
    tri_residual: float | None = None


class _Fp64Workspace:
    """Every device buffer one FP64-mode refinement needs, allocated once."""

    def __init__(self, n, device):
        self.n = n
        self.q = ZPlanar.empty(n, device=device)
        self.q_next = ZPlanar.empty(n, device=device)
        self.p = ZPlanar.empty(n, device=device)        # Q^H A
        self.that = ZPlanar.empty(n, device=device)     # (Q^H A) Q
        self.y = ZPlanar.empty(n, device=device)        # Q^H Q - I
        self.sigma = ZPlanar.empty(n, device=device)
        self.t_lp = lp_empty(n, device=device)
        self.e_lp = lp_empty(n, device=device)
        self.l_lp = lp_empty(n, device=device)
        self.w_lp = lp_empty(n, device=device)
        self.y_lp = lp_empty(n, device=device)
        self.yw = lp_empty(n, device=device)
        self.w2 = lp_empty(n, device=device)
        self.w3 = lp_empty(n, device=device)
        self.w2y = None
        self.w2yw = None
        self.scal = torch.zeros(8, dtype=torch.float64, device=device)  # norm_a, norm_e, norm_y, norm_w
        self.in_flags = torch.zeros(1, dtype=torch.int32, device=device)  # deferred input checks (A 1, Q^ 2)
        self.perm_ws = torch.empty(_lib.load().sr_phase_perm_workspace_bytes(n), dtype=torch.uint8, device=device)
        self.perm_row = torch.empty(n, dtype=torch.int32, device=device)
        red = _lib.load().sr_reduce_workspace_bytes()
        self.red = [torch.zeros(red, dtype=torch.uint8, device=device) for _ in range(4)]
        self.solver = SolverWorkspace(n, torch.complex64, device)
        self.staging = None
        self.inputs = None
        self.device = device

    def host_staging(self):
        """Interleaved complex128 device staging buffers for Q and T when the
        result goes to host tensors (allocated on first use)."""
        if self.staging is None:
            self.staging = tuple(torch.empty((self.n, self.n), dtype=torch.complex128, device=self.device)
                                 for _ in range(2))
        return self.staging

    def host_inputs(self, real_a):
        """Device landing buffers for host inputs (Q^ planar, A planar real or
        complex), kept across calls so an end-to-end call allocates nothing."""
        if self.inputs is None:
            self.inputs = {}
        key = "a_real" if real_a else "a_cplx"
        if "qhat" not in self.inputs:
            self.inputs["qhat"] = ZPlanar.empty(self.n, device=self.device)
        if key not in self.inputs:
            self.inputs[key] = ZPlanar.empty(self.n, device=self.device, real=real_a)
        return self.inputs["qhat"], self.inputs[key]

    def ptr(self, i):
        return self.scal.data_ptr() + 8 * i

    def fro_norm(self, x):
        """||x||_F of a ZPlanar (deterministic reduction; one host sync)."""
        _lib.call("sr_fro_norm_f64", self.n, self.n, x.re_ptr(), x.im_ptr(), x.ld, self.ptr(5),
                  self.red[0].data_ptr(), self.red[0].numel(), _stream())
        return float(self.scal[5].cpu())


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _finite_flag(m, flags, bit):
    """flags |= bit if the planar matrix m has a non-finite entry (one pass in
    libsr, no host sync; read with the caller's next sync)."""
    _lib.call("sr_finite_flag_f64", m.rows, m.cols, m.re_ptr(), m.im_ptr(), m.ld, flags.data_ptr(), bit, _stream())


def _coerce(x, device, flags=None, bit=1):
    """_coerce_hp (refine.py:341-350): exact embed, square + finite checks.
    With `flags`, the finiteness check is only launched (flags |= bit on the
    device) and the caller raises at its next host sync; without, it is read
    at once."""
    if isinstance(x, ZPlanar):
        m = x
    else:
        if isinstance(x, np.ndarray):
            if x.ndim != 2:
                raise ValueError("expected a 2-d array")
        m = ZPlanar.from_any(x, device=device)
    if m.rows != m.cols:
        raise ValueError("refinement needs a square matrix")
    if flags is None:
        f = torch.zeros(1, dtype=torch.int32, device=m.re_buf.device)
        _finite_flag(m, f, 1)
        if int(f.item()):
            raise ValueError("input matrix has non-finite entries")
    else:
        _finite_flag(m, flags, bit)
    return m


def _raise_nonfinite(flags_value):
    """The deferred finiteness checks: A (bit 1) is validated before Q^ (bit 2),
    like the reference's two _coerce_hp calls (refine.py:374-375)."""
    if flags_value & 3:
        raise ValueError("input matrix has non-finite entries")


def _is_host_matrix(x):
    return isinstance(x, np.ndarray) or (isinstance(x, torch.Tensor) and x.device.type == "cpu")


def _host_tensor(x):
    if isinstance(x, np.ndarray):
        if x.ndim != 2:
            raise ValueError("expected a 2-d array")
        x = torch.from_numpy(np.ascontiguousarray(x))
    if x.dim() != 2:
        raise ValueError("expected a 2-d array")
    return x


def _h2d_planar(x, dst, landing):
    """Copy a host (n, n) matrix, real or complex, C or Fortran order, into
    the planar device matrix dst: one contiguous H2D of its storage into
    the interleaved complex128 landing buffer, then a de-interleave (and,
    for Fortran order, a transpose) on the device."""
    n = x.shape[0]
    if x.is_contiguous():
        src, transposed = x, False
    elif x.t().is_contiguous():  # Fortran order (LAPACK outputs): copy the storage as is
        src, transposed = x.t(), True
    else:
        src, transposed = x.contiguous(), False
    if src.is_complex():
        src = src.to(torch.complex128) if src.dtype != torch.complex128 else src
        stage = landing
    else:
        src = src.to(torch.float64) if src.dtype != torch.float64 else src
        stage = torch.view_as_real(landing).view(-1)[: n * n].view(n, n)
    stage.copy_(src, non_blocking=True)
    view = stage.t() if transposed else stage
    if src.is_complex():
        dst.re_buf[:, :n].copy_(view.real)
        dst.im_buf[:, :n].copy_(view.imag)
    else:
        dst.re_buf[:, :n].copy_(view)
        if dst.im_buf is not None:
            dst.im_buf.zero_()
    if dst.ld != n:
        dst.re_buf[:, n:].zero_()
        if dst.im_buf is not None:
            dst.im_buf[:, n:].zero_()
    return dst


def _upload_qhat(x, dst, landing, flags):
    """_coerce_hp (refine.py:341-350) of a host Q^ into the workspace's planar
    buffer (the landing buffer is the workspace's result staging, free until
    the first measurement); the finiteness check runs on the device into
    flags (bit 2), read with the entry step's first sync."""
    x = _host_tensor(x)
    if x.shape[0] != x.shape[1]:
        raise ValueError("refinement needs a square matrix")
    _h2d_planar(x, dst, landing)
    _finite_flag(dst, flags, 2)
    return dst


class _AsyncUpload:
    """A host matrix copied to the device on a side stream, so the copy
    overlaps the entry step (A is first needed by the first measurement);
    the finiteness check (_coerce_hp, refine.py:341-350) is evaluated on the
    device and raised as soon as A is needed."""

    def __init__(self, x, device, dst=None, landing=None):
        x = _host_tensor(x)
        rows, cols = x.shape
        if rows != cols:
            raise ValueError("refinement needs a square matrix")
        main = torch.cuda.current_stream(device)
        self.m = dst if dst is not None else ZPlanar.empty(rows, cols, device=device, real=not x.is_complex())
        self.stream = torch.cuda.Stream(device=device)
        self.stream.wait_stream(main)
        with torch.cuda.stream(self.stream):
            if landing is not None:
                _h2d_planar(x, self.m, landing)
            else:
                ZPlanar.fill_from(self.m, x)
            self.flags = torch.zeros(1, dtype=torch.int32, device=device)
            _finite_flag(self.m, self.flags, 1)
            self.ready = torch.cuda.Event()
            self.ready.record(self.stream)
        self.host = x  # pinned source stays alive until the copy has run

    def check(self):
        # the flag is computed on the upload stream: order the read after it
        torch.cuda.current_stream(self.flags.device).wait_event(self.ready)
        if int(self.flags.item()):
            raise ValueError("input matrix has non-finite entries")


def _newton_schulz_entry(qhat, ws, prod, a_upload=None):
    """newton_schulz_step (orthogonal.py:153-169): guard ||Q^||_2 < sqrt(3)
    by lp power iteration, then Q = Q^ (3I - Q^H Q^) / 2 in hp."""
    n = ws.n
    _lib.call("sr_downcast_c64", n, n, qhat.re_ptr(), qhat.im_ptr(), qhat.ld, ws.y_lp.data_ptr(),
              ws.y_lp.shape[1], _stream())
    est = spectral_norm_estimate(ws.y_lp, n)
    _raise_nonfinite(int(ws.in_flags.item()))  # the GPU is idle here: a 4-byte read
    if not est < math.sqrt(3.0):
        if a_upload is not None:  # the reference validates A before the entry step
            a_upload.check()
        raise NormTooLarge("spectral norm estimate %.6f is not below sqrt(3)" % est)
    prod.entry(qhat)


def _phase_permutation(q, ws=None):
    """_phase_permutation (refine.py:172-189): perm with q[perm[j], j] the only
    nonzero of column j and of its row, each of exactly unit modulus; else None.
    The O(n^2) pattern scan is one libsr pass (sr_phase_perm_scan_f64) and a
    4-byte read; only a permutation pattern goes on to the O(n) exact
    unit-modulus check on the host."""
    n = q.cols
    dev = q.re_buf.device
    if ws is not None and getattr(ws, "n", None) == n:
        scratch, row = ws.perm_ws, ws.perm_row
    else:
        scratch = torch.empty(_lib.load().sr_phase_perm_workspace_bytes(n), dtype=torch.uint8, device=dev)
        row = torch.empty(n, dtype=torch.int32, device=dev)
    status = row.new_zeros(1)
    _lib.call("sr_phase_perm_scan_f64", n, q.re_ptr(), q.im_ptr(), q.ld, row.data_ptr(), status.data_ptr(),
              scratch.data_ptr(), scratch.numel(), _stream())
    if not int(status.item()):
        return None
    perm = row.long()
    cols = torch.arange(n, device=dev)
    zr = q.re[perm, cols].double().cpu().numpy()
    zi = (q.im[perm, cols] if q.im is not None else torch.zeros_like(q.re[perm, cols])).cpu().numpy()
    from fractions import Fraction
    for x, y in zip(zr.tolist(), zi.tolist()):
        if Fraction(x) ** 2 + Fraction(y) ** 2 != 1:
            return None
    return perm


def _structural_triangle(a, q, perm, symmetric=False):
    """_permuted_part_is_zero + _exact_similarity_triangle (refine.py:192-220):
    if A[perm][:, perm] is exactly upper triangular (diagonal when symmetric),
    T = conj(q_p) A_pp q_p entrywise (no products); else None."""
    sub_re = a.re[perm][:, perm]
    nz = sub_re != 0
    if a.im is not None:
        nz = nz | (a.im[perm][:, perm] != 0)
    if bool(torch.tril(nz, -1).any()) or (symmetric and bool(torch.triu(nz, 1).any())):
        return None
    cols = torch.arange(q.cols, device=perm.device)
    ph = torch.complex(q.re[perm, cols], q.im[perm, cols] if q.im is not None else torch.zeros_like(sub_re[0]))
    sub = torch.complex(sub_re, a.im[perm][:, perm] if a.im is not None else torch.zeros_like(sub_re))
    t = torch.triu(ph.conj()[:, None] * sub * ph[None, :])
    if symmetric:  # the real diagonal only (refine.py:214-219)
        t = torch.diag(torch.diagonal(t).real).to(t.dtype)
    return t


def _quarter_phases(q, perm):
    """The phases of a phase-permutation Q when all are +-1 or +-i (then every
    product with Q or Q^H is exact data movement), else None."""
    if perm is None:
        return None
    cols = torch.arange(q.cols, device=perm.device)
    re = q.re[perm, cols]
    im = q.im[perm, cols] if q.im is not None else torch.zeros_like(re)
    ok = (((re.abs() == 1) & (im == 0)) | ((re == 0) & (im.abs() == 1))).all()
    return torch.complex(re, im) if bool(ok) else None


def _permuted_similarity(ph, perm, re, im):
    """conj(ph_i) X[perm_i, perm_j] ph_j for one planar FP64 pair (exact for
    quarter phases: sign flips and re/im swaps)."""
    x = torch.complex(re[perm][:, perm], im[perm][:, perm] if im is not None else torch.zeros_like(re))
    return ph.conj()[:, None] * x * ph[None, :]


def _exact_measure(a, ph, perm, that, y):
    """T^ = Q^H A Q and Y = Q^H Q - I = 0 for Q = P diag(ph), ph in {+-1, +-i}
    (refine.py:259,265): the reference's dd GEMMs are exact on such a Q, and
    so is this — whereas an Ozaki product would resolve A's entries only to
    2^-beta of their column maximum (the 1e-200 separations of
    test_refine.py:266-287).  a / that / y: ZPlanar, or DDPlanar (both pairs)."""
    pairs = ((a.hi, that.hi, y.hi), (a.lo, that.lo, y.lo)) if hasattr(a, "hi") else ((a, that, y),)
    n = that.cols
    for src, dst, yy in pairs:
        t = _permuted_similarity(ph, perm, src.re, src.im)
        dst.re_buf[:, :n].copy_(t.real)
        dst.im_buf[:, :n].copy_(t.imag)
        yy.re_buf.zero_()
        yy.im_buf.zero_()
    _counters["hp_calls"] += 3  # the reference's three logical products (refine.py:259,265)


class _HostResult:
    """Device->host delivery of the result into caller-provided pinned host
    tensors (refine_template(out=(q_host, t_host))):
    the Q each measurement sees is copied to pinned host memory on a side
    stream while that measurement runs — the last one is the returned Q
    whenever the loop ends without a further update (convergence with the
    skip rule, the config-3 case) — and T is copied at the end."""

    def __init__(self, n, device, q_host, t_host, bufs):
        for h in (q_host, t_host):
            if not (isinstance(h, torch.Tensor) and h.device.type == "cpu" and h.dtype == torch.complex128
                    and tuple(h.shape) == (n, n) and h.is_contiguous()):
                raise ValueError("out must be two contiguous (n, n) complex128 CPU tensors")
        self.n = n
        self.stream = torch.cuda.Stream(device=device)
        self.buf, self.tbuf = bufs  # device staging for Q and T (kept in the workspace)
        self.done = torch.cuda.Event()
        self.q_host, self.t_host = q_host, t_host
        self.copied_version = -1
        self.started = False
        self.t_copied = False

    def copy_q(self, q, version):
        main = torch.cuda.current_stream()
        if self.started:
            main.wait_event(self.done)  # the previous D2H has left buf
        q.to_complex(out=self.buf)
        ready = torch.cuda.Event()
        ready.record(main)
        self.stream.wait_event(ready)
        with torch.cuda.stream(self.stream):
            self.q_host.copy_(self.buf, non_blocking=True)
            self.done.record(self.stream)
        self.started = True
        self.copied_version = version

    def copy_t(self, t):
        t.to_complex(out=self.tbuf)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream())
        self.stream.wait_event(ready)
        with torch.cuda.stream(self.stream):
            self.t_host.copy_(self.tbuf, non_blocking=True)
            self.done.record(self.stream)
        self.t_copied = True

    def finish(self, q, version, t):
        if self.copied_version != version:
            self.copy_q(q, version)
        if not self.t_copied:
            self.t_host.copy_(t.to_complex(out=self.tbuf), non_blocking=True)
        self.done.synchronize()
        torch.cuda.current_stream().synchronize()
        return self.q_host, self.t_host


def _finalize_t(ws, symmetric, st):
    """T = triu(T^) in place (real diagonal parts only when symmetric); idempotent."""
    _lib.call("sr_triu_inplace_f64", ws.n, ws.that.re_ptr(), ws.that.im_ptr(), ws.that.ld, st)
    if symmetric:  # T keeps its real parts (refine.py:435-436)
        ws.that.im.zero_()


def _run_fp64(a, qhat, cfg, ws, symmetric=False, host=None, a_upload=None):
    """_run (refine.py:223-329) with hp = FP64, lp = complex64.  symmetric
    (refine_symmetric): the defect is the full off-diagonal part of Q^H A Q
    and the solve is the entrywise diagonal correction."""
    n = a.rows
    st = _stream()
    hp0 = _counters["hp_calls"]
    _mark("start")
    prod = products.make(cfg.gemm, ws, a)
    if cfg.restore_full_sigma:
        products.ensure_full_sigma_buffers(ws)
    _mark("setup")
    _newton_schulz_entry(qhat, ws, prod, a_upload)
    _mark("entry")
    if a_upload is not None:  # A's host->device copy ran on a side stream during the entry
        torch.cuda.current_stream().wait_event(a_upload.ready)
        a_upload.check()
    _lib.call("sr_fro_norm_f64", n, n, a.re_ptr(), a.im_ptr(), a.ld, ws.ptr(0), ws.red[0].data_ptr(),
              ws.red[0].numel(), st)
    history = []
    perm = _phase_permutation(ws.q, ws)
    if perm is not None:
        t_exact = _structural_triangle(a, ws.q, perm, symmetric)
        if t_exact is not None:
            # exactly unitary Q, exactly triangular Q^H A Q: zero iterations
            # beyond the entry check (refine.py:239-252)
            history.append((0.0, 0.0))
            q_out = ws.q.to_complex()
            if host is not None:
                host.q_host.copy_(q_out)
                host.t_host.copy_(t_exact)
                q_out, t_exact = host.q_host, host.t_host
            pair = SchurPair(q=q_out, t=t_exact, ortho_residual=0.0, tri_residual=0.0)
            report = RefineReport(iterations=0, residual_history=history,
                                  hp_matmul_count=_counters["hp_calls"] - hp0, clipped_total=0,
                                  status=RefineStatus.CONVERGED, wall_time=0.0)
            return pair, report
    clipped_total = 0
    skip_fired = False
    detail = ""
    status = RefineStatus.MAX_ITERS
    iterations = cfg.max_iters
    streak = 0
    tol = None
    q_version = 0
    ph = _quarter_phases(ws.q, perm)
    for it in range(1, cfg.max_iters + 1):
        if host is not None:  # this Q is the result if the loop stops without another update
            host.copy_q(ws.q, q_version)
        # T^ = (Q^H A) Q; split + lp downcast + ||E||; Y = Q^H Q - I; ||Y||
        if ph is not None:  # Q a signed permutation: exact data movement (_exact_measure)
            _exact_measure(a, ph, perm, ws.that, ws.y)
        else:
            prod.measure(a)
        _mark("measure")
        _lib.call("sr_split_lp_c64", n, ws.that.re_ptr(), ws.that.im_ptr(), ws.that.ld, ws.t_lp.data_ptr(),
                  ws.e_lp.data_ptr(), ws.t_lp.shape[1], ws.ptr(1), ws.red[1].data_ptr(), ws.red[1].numel(), st)
        _lib.call("sr_fro_norm_f64", n, n, ws.y.re_ptr(), ws.y.im_ptr(), ws.y.ld, ws.ptr(2),
                  ws.red[2].data_ptr(), ws.red[2].numel(), st)
        if symmetric:  # + ||striu(T^)||: the full off-diagonal defect (refine.py:130-131)
            _lib.call("sr_striu_norm_f64", n, ws.that.re_ptr(), ws.that.im_ptr(), ws.that.ld, ws.ptr(6),
                      ws.red[1].data_ptr(), ws.red[1].numel(), st)
        _mark("split_norms")
        s = ws.scal[:7].cpu()  # sync 1
        norm_a, norm_e, norm_y = float(s[0]), float(s[1]), float(s[2])
        if symmetric:
            norm_e = math.hypot(norm_e, float(s[6]))
        if tol is None:
            tol = cfg.tol_factor * n * U_FP64 * norm_a
            # row 0: entry state measured in FP64 (see oracle/refine_fp64.py)
            history.append((norm_e, norm_y))
        history.append((norm_e, norm_y))
        if not (math.isfinite(norm_e) and math.isfinite(norm_y)):
            status, iterations = RefineStatus.NON_FINITE, it
            detail = "iteration %d: residuals became non-finite" % it
            if cfg.clip_threshold is None:
                detail += "; " + _CLIP_HINT
            break
        converged = norm_e <= tol
        if converged and host is not None:
            # this measurement's T is the result: its device->host copy overlaps the solve
            _finalize_t(ws, symmetric, st)
            host.copy_t(ws.that)
        # lp solve + W = L - L^H + ||W|| + finiteness
        ws.solver.clipped.zero_()
        ws.solver.flags.zero_()
        if symmetric:
            clip = 0.0 if cfg.clip_threshold is None else float(cfg.clip_threshold)
            _lib.call("sr_diag_correction_c64", n, ws.t_lp.data_ptr(), ws.e_lp.data_ptr(), ws.t_lp.shape[1],
                      ws.l_lp.data_ptr(), clip, ws.solver.clipped.data_ptr(), ws.solver.flags.data_ptr(), st)
        else:
            solve_lp_device(ws.t_lp, ws.e_lp, ws.l_lp, n, cfg.clip_threshold, ws.solver, st)
        _mark("solve")
        _lib.call("sr_skew_c64", n, ws.l_lp.data_ptr(), ws.l_lp.shape[1], ws.w_lp.data_ptr(), ws.ptr(3),
                  ws.solver.flags.data_ptr(), ws.red[3].data_ptr(), ws.red[3].numel(), st)
        _mark("skew")
        norm_w = float(ws.scal[3].cpu())  # sync 2
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
        skip = (converged and cfg.skip_final_ortho and norm_y <= 10.0 * n * U_FP64
                and norm_w <= math.sqrt(U_FP64))
        if not skip:
            prod.update(cfg.restore_full_sigma,
                        sigma_bound=products.sigma_prime_bound(norm_y, norm_w, cfg.restore_full_sigma),
                        norm_y=norm_y, norm_w=norm_w)
            q_version += 1
            if ph is not None:  # still a signed permutation (W = 0: every correction clipped)?
                perm = _phase_permutation(ws.q, ws)
                ph = _quarter_phases(ws.q, perm)
            _mark("update")
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
    _finalize_t(ws, symmetric, st)
    last_e, last_y = history[-1]
    if host is not None:
        q_out, t_out = host.finish(ws.q, q_version, ws.that)
    else:
        q_out, t_out = ws.q.to_complex(), ws.that.to_complex()
    _mark("result")
    pair = SchurPair(q=q_out, t=t_out, ortho_residual=last_y, tri_residual=last_e)
    report = RefineReport(iterations=iterations, residual_history=history,
                          hp_matmul_count=_counters["hp_calls"] - hp0, clipped_total=clipped_total,
                          status=status, wall_time=0.0, skip_fired=skip_fired, detail=detail)
    return pair, report


_WS_CACHE = {}

PHASES = None  # list of (label, cuda event) while phase profiling is on (tools/time_refine.py)


def _mark(label):
    if PHASES is not None:
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        PHASES.append((label, ev))


def _workspace(n, device):
    key = (n, str(device))
    ws = _WS_CACHE.get(key)
    if ws is None:
        _WS_CACHE.clear()
        ws = _WS_CACHE[key] = _Fp64Workspace(n, device)
    return ws


def refine_template(a, qhat, cfg=None, device=None, out=None):
    """Refine a user-supplied candidate Q toward a Schur pair of A
    (refine.py:357-380).  a, qhat: numpy arrays, torch tensors (any device)
    or ZPlanar device matrices; real A is kept real.  Returns
    (SchurPair, RefineReport) with q, t as complex128 CUDA tensors, or (FP64
    mode, out=(q_host, t_host): two (n, n) complex128 CPU tensors, pinned for
    asynchronous copies) written into those host tensors — like the
    reference's host DDMatrix result — with Q's device->host copy overlapped
    with the final measurement."""
    cfg = RefineConfig() if cfg is None else cfg
    if cfg.ortho is not OrthoStrategy.NEWTON_SCHULZ:
        raise NotImplementedError("QR retraction is not on the B200 path (no CPU fallback)")
    if not torch.cuda.is_available():
        raise RuntimeError("refine_template needs a CUDA device (no CPU fallback)")
    device = torch.device("cuda") if device is None else torch.device(device)
    t0 = time.perf_counter()
    _mark("call")
    if cfg.precision == "dd":
        if out is not None:
            raise ValueError("out=(q_host, t_host) is the FP64-mode host delivery; dd mode returns DDPlanar results")
        from . import dd_refine
        a = dd_refine.coerce_dd(a, device)
        qhat = dd_refine.coerce_dd(qhat, device)
        if a.shape != qhat.shape:
            raise ValueError("matrix and candidate shapes differ")
        pair, report = dd_refine.run_dd(a, qhat, cfg, device)
        torch.cuda.current_stream().synchronize()
        report.wall_time = time.perf_counter() - t0
        return pair, report
    ws = None
    # double-double operands in FP64 mode: their binary64 rounding (the hi cells)
    a, qhat = (x.to_lp() if hasattr(x, "to_lp") else x for x in (a, qhat))
    if _is_host_matrix(qhat) and _is_host_matrix(a):
        # end to end from host memory: every device buffer comes from the workspace
        qh, ah = _host_tensor(qhat), _host_tensor(a)
        if qh.shape[0] != qh.shape[1] or ah.shape[0] != ah.shape[1]:
            raise ValueError("refinement needs a square matrix")
        if ah.shape != qh.shape:
            raise ValueError("matrix and candidate shapes differ")
        ws = _workspace(qh.shape[0], device)
        ws.in_flags.zero_()
        q_dst, a_dst = ws.host_inputs(real_a=not ah.is_complex())
        qhat = _upload_qhat(qh, q_dst, ws.host_staging()[0], ws.in_flags)
        # A's H2D lands in T's result staging buffer (dead once copied into a_dst;
        # T is first staged after the main stream waited for the upload)
        a_upload = _AsyncUpload(ah, device, dst=a_dst, landing=ws.host_staging()[1])
        a = a_upload.m
    else:
        # both square and of one size: the finiteness checks are deferred to the
        # entry step's first host read (ws.in_flags); otherwise _coerce raises now
        shapes = [tuple(x.shape) if hasattr(x, "shape") else None for x in (a, qhat)]
        n_in = shapes[0][0] if shapes[0] is not None and len(shapes[0]) == 2 else 0
        ws = _workspace(n_in, device) if (n_in > 0 and shapes[0] == shapes[1] == (n_in, n_in)) else None
        flags = None
        if ws is not None:
            ws.in_flags.zero_()
            flags = ws.in_flags
        a_upload = None
        if _is_host_matrix(a):
            a_upload = _AsyncUpload(a, device)
            a = a_upload.m
        else:
            a = _coerce(a, device, flags, 1)
        qhat = _coerce(qhat, device, flags, 2)
    if a.shape != qhat.shape:
        raise ValueError("matrix and candidate shapes differ")
    if qhat.is_real:
        qhat = ZPlanar.from_any(qhat.re, device=device, force_complex=True)
    if True:
        ws = _workspace(a.rows, device) if ws is None else ws
        host = _HostResult(a.rows, device, *out, bufs=ws.host_staging()) if out is not None else None
        pair, report = _run_fp64(a, qhat, cfg, ws, host=host, a_upload=a_upload)
    torch.cuda.current_stream().synchronize()
    report.wall_time = time.perf_counter() - t0
    return pair, report


VERIFY_DD_BETA = 106  # every dd entry within 2^-0 of its row maximum keeps 106 bits (30 moduli)


class VerifyResiduals(NamedTuple):
    """refine.py:105-108."""

    ortho_residual: float
    tri_residual: float
    similarity_residual: float


def verify_pair(a, pair, device=None, precision="dd"):
    """verify_pair (refine.py:456-476) on the GPU: the three quality residuals
    (||Q^H Q - I||_F, ||stril(Q^H A Q)||_F, ||T - Q^H A Q||_F) of a Schur pair,
    measured from scratch.  precision "dd" (the reference's): the products as
    Ozaki-II double-double products (beta = 102, dd in and out), T - Q^H A Q
    subtracted in dd; "fp64": FP64 Ozaki-II products.  a, pair.q, pair.t: any
    matrix refine_template accepts (numpy, torch, 4-plane dd).  Returns
    VerifyResiduals (floats)."""
    from . import dd_refine, ozaki
    from .matrix import DDPlanar
    if precision not in ("dd", "fp64"):
        raise ValueError("precision must be 'dd' or 'fp64'")
    device = torch.device("cuda") if device is None else torch.device(device)
    if precision == "dd":
        A = dd_refine.coerce_dd(a, device)
        Q = dd_refine.coerce_dd(pair.q, device)
        T = dd_refine.coerce_dd(pair.t, device)
        n = A.rows
        if Q.rows != n or T.rows != n:
            raise ValueError("pair dimensions do not match the matrix")
        pl = ozaki.plan(n, VERIFY_DD_BETA, VERIFY_DD_BETA)
        mk = lambda: DDPlanar.empty(n, device=device)  # noqa: E731
    else:
        A = _coerce(a, device)
        Q = ZPlanar.from_any(pair.q, device=device, force_complex=True)
        T = ZPlanar.from_any(pair.t, device=device, force_complex=True)
        n = A.rows
        if Q.rows != n or T.rows != n:
            raise ValueError("pair dimensions do not match the matrix")
        pl = ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA)
        mk = lambda: ZPlanar.empty(n, device=device)  # noqa: E731
    eqh = ozaki.Encoded(n, n, 2, pl.beta_a, pl.nmod, device)
    eq = ozaki.Encoded(n, n, 3, pl.beta_b, pl.nmod, device)
    ozaki.encode_dual(Q, n, n, pl, eqh, eq)
    res = ozaki.ResidueBuffer(n, n, pl.nmod, device)
    g = mk()
    ozaki.gemm_residues(eqh, eq, pl, res, lower_only=True)
    ozaki.decode(res, eqh, eq, pl, g, shift=-1.0, hermitian=True)        # Q^H Q - I
    eb_a = ozaki.encode(A, n, n, "b", pl)
    p = mk()
    ozaki.gemm_residues(eqh, eb_a, pl, res)
    ozaki.decode(res, eqh, eb_a, pl, p)                                   # Q^H A
    ea_p = ozaki.encode(p, n, n, "a", pl)
    that = mk()
    ozaki.gemm_residues(ea_p, eq, pl, res)
    ozaki.decode(res, ea_p, eq, pl, that)                                 # (Q^H A) Q

    def planes(x):  # (re, im) float64 values; dd: hi + lo rounded once
        if precision == "dd":
            return x.hi.re + x.lo.re, x.hi.im + x.lo.im
        return x.re, x.im

    def fro(re, im):
        return float(torch.sqrt((re * re).sum() + (im * im).sum()))

    gr, gi = planes(g)
    tr, ti = planes(that)
    low = torch.tril(torch.ones(n, n, dtype=torch.bool, device=device), -1)
    if precision == "dd":  # T - T^ in dd: the hi parts cancel exactly (Sterbenz) for a refined pair
        dr = (T.hi.re - that.hi.re) + (T.lo.re - that.lo.re)
        di = (T.hi.im - that.hi.im) + (T.lo.im - that.lo.im)
    else:
        dr, di = T.re - that.re, T.im - that.im
    return VerifyResiduals(ortho_residual=fro(gr, gi), tri_residual=fro(tr * low, ti * low),
                           similarity_residual=fro(dr, di))