"""The matrix products of one FP64-mode refinement, two implementations.

Every product the loop needs (refine.py:259,265 and orthogonal.py:167-201):
  entry    Q = (Q^ (3I - Q^H Q^)) / 2                    (2 hp products)
  measure  P = Q^H A, T^ = P Q, Y = Q^H Q - I            (3 hp products)
  update   YW, W^2, W^3 (lp), Sigma (hp sum), Q S / 2    (3 lp + 1 hp product;
           the Ozaki path forms W^2 and X W = YW - W^2 - W^3, X = Y - W - W^2:
           two lp products, the first Hermitian)

OzakiProducts (default) runs them as Ozaki-II emulated products on the int8
tensor cores (ozaki.py, csrc/oz_gemm.cu): exact integer products, so the
stril(Q^H A Q) measurement noise does not grow with n, and the update is
formed as Q + Q S'/2 with S' = S - 2I (the same matrix as Q S / 2,
with one rounding instead of a K-long accumulation).  DmmaProducts runs
them on the FP64 DMMA pipe (csrc/zgemm_f64.cu) and the FP32 SIMT lp GEMM
(csrc/cgemm_c64.cu); it is kept as the native-FP64 comparison point.
"""
import os

import torch

from . import _lib, ozaki
from .matmul import _counters, matmul_hp, matmul_lp
from .matrix import ZPlanar, lp_empty


def _stream():
    return torch.cuda.current_stream().cuda_stream


def _sigma(ws, restore_full_sigma, with_identity, fused=False, drop_lp=False):
    """S (or S' = S - 2I) from W, Y and the lp products; fused: ws.yw holds
    X W = YW - W^2 - W^3 (X = Y - W - W^2) and W^2, W^3 are not separate;
    drop_lp (fused only): that product is negligible, S' = 2W - Y."""
    n = ws.n
    w2y = w2yw = None
    if restore_full_sigma:
        w2y, w2yw = ws.w2y.data_ptr(), ws.w2yw.data_ptr()
    w2, w3 = (None, None) if fused else (ws.w2.data_ptr(), ws.w3.data_ptr())
    _lib.call("sr_sigma_merged_f64", n, n, ws.w_lp.data_ptr(), ws.y.re_ptr(), ws.y.im_ptr(), ws.y.ld,
              None if (fused and drop_lp) else ws.yw.data_ptr(), w2, w3, w2y, w2yw, ws.w_lp.shape[1],
              ws.sigma.re_ptr(), ws.sigma.im_ptr(), ws.sigma.ld, 1 if with_identity else 0, _stream())


def _downcast_y(ws):
    n = ws.n
    _lib.call("sr_downcast_c64", n, n, ws.y.re_ptr(), ws.y.im_ptr(), ws.y.ld, ws.y_lp.data_ptr(),
              ws.y_lp.shape[1], _stream())


class DmmaProducts:
    name = "dmma"

    def __init__(self, ws, a):
        self.ws = ws

    def entry(self, qhat):
        ws = self.ws
        n = ws.n
        g = matmul_hp(qhat, qhat, trans_a=True, out=ws.y)
        _lib.call("sr_sigma_ns_f64", n, g.re_ptr(), g.im_ptr(), g.ld, ws.sigma.re_ptr(), ws.sigma.im_ptr(),
                  ws.sigma.ld, _stream())
        matmul_hp(qhat, ws.sigma, alpha=0.5, out=ws.q)

    def measure(self, a):
        ws = self.ws
        matmul_hp(ws.q, a, trans_a=True, out=ws.p)
        matmul_hp(ws.p, ws.q, out=ws.that)
        matmul_hp(ws.q, ws.q, trans_a=True, diag_shift=-1.0, out=ws.y)

    def update(self, restore_full_sigma, sigma_bound=None, norm_y=None, norm_w=None):
        ws = self.ws
        n = ws.n
        _downcast_y(ws)
        matmul_lp(ws.y_lp, ws.w_lp, n, n, n, out=ws.yw)
        matmul_lp(ws.w_lp, ws.w_lp, n, n, n, out=ws.w2)
        matmul_lp(ws.w2, ws.w_lp, n, n, n, out=ws.w3)
        if restore_full_sigma:
            matmul_lp(ws.w2, ws.y_lp, n, n, n, out=ws.w2y)
            matmul_lp(ws.w2y, ws.w_lp, n, n, n, out=ws.w2yw)
        _sigma(ws, restore_full_sigma, True)
        matmul_hp(ws.q, ws.sigma, alpha=0.5, out=ws.q_next)
        ws.q, ws.q_next = ws.q_next, ws.q


class OzakiProducts:
    """All products on the int8 tensor cores; encodings are reused across the
    products that share an operand (Q^H feeds P and Y, Q feeds T^ and Y, the
    constant A is encoded once per refinement, W once per update)."""

    name = "ozaki"

    def __init__(self, ws, a, gauss=True):
        """gauss (default): Gaussian-CRT plans — every complex product is two
        real products per modulus (one for the Hermitian Q^H Q and W^2), and
        one encoding of Q serves as Q (B role) and Q^H (A role, planes
        swapped); gauss=False: the (re, im) planes, four real products."""
        self.ws = ws
        self.gauss = gauss
        n = ws.n
        dev = ws.q.re_buf.device
        self.hp = ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA, gauss)
        self.lp = ozaki.plan(n, ozaki.LP_BETA, ozaki.LP_BETA, gauss)
        # the measurement's plans: Q^H Q (hq), P = Q^H A (hp_p), T^ = P Q (hp_t);
        # with Gaussian planes Q is encoded once, at beta HP_BETA_Q
        bq = ozaki.HP_BETA_Q if gauss else ozaki.HP_BETA
        self.hq = ozaki.plan(n, bq, bq, gauss)
        self.hp_p = ozaki.plan(n, bq, ozaki.HP_BETA, gauss)
        self.hp_t = ozaki.plan(n, ozaki.HP_BETA, bq, gauss)
        hp, lp = self.hp, self.lp
        bpl = 2 if gauss else 3
        self.ea_qh = None if gauss else ozaki.Encoded(n, n, 2, hp.beta_a, hp.nmod, dev)   # Q^H, A role
        self.ea_x = ozaki.Encoded(n, n, 2, hp.beta_a, hp.nmod, dev)    # P or Q, A role
        self.eb_q = ozaki.Encoded(n, n, bpl, hp.beta_b, hp.nmod, dev)  # Q, B role
        self.eb_s = ozaki.Encoded(n, n, bpl, hp.beta_b, hp.nmod, dev)  # Sigma' / Y', B role
        self.res = ozaki.ResidueBuffer(n, n, hp.nmod, dev)
        self.la = ozaki.Encoded(n, n, 2, lp.beta_a, lp.nmod, dev)      # Y_lp / W / W^2, A role
        self.lb = ozaki.Encoded(n, n, bpl, lp.beta_b, lp.nmod, dev)    # W, B role
        self.lres = ozaki.ResidueBuffer(n, n, lp.nmod, dev)
        # the constant matrix A, B role (real A keeps one plane), encoded at the
        # first measurement so an asynchronous upload of A overlaps the entry step
        self.a = a
        self.eb_a = None
        # W exactly skew-Hermitian (W = L - L^H, sr_skew_c64): W^2 / W^3 on the
        # lower tiles; False (orthogonal.merged_update of a general W): full products
        self.w_skew = True

    def _hp(self, ea, eb, out, hermitian=False, pl=None, **kw):
        pl = ozaki.fit_plan(pl or self.hp, ea, eb)  # fewest moduli the operands' norms allow
        ozaki.gemm_residues(ea, eb, pl, self.res, lower_only=hermitian)
        ozaki.decode(self.res, ea, eb, pl, out, hermitian=hermitian, **kw)
        _counters["hp_calls"] += 1

    def _lp(self, ea, eb, out, hermitian=False):
        self._lp_with(self.lp, ea, eb, out, hermitian)

    def _lp_with(self, pl, ea, eb, out, hermitian=False, alpha=1.0):
        pl = ozaki.fit_plan(pl, ea, eb)
        ozaki.gemm_residues(ea, eb, pl, self.lres, lower_only=hermitian if hermitian == "skew" else bool(hermitian))
        ozaki.decode(self.lres, ea, eb, pl, out, alpha=alpha, hermitian=hermitian)
        _counters["lp_calls"] += 1

    def _correction_plan(self, bound):
        """Plan for X S with a small S (||S||_F <= bound) added to an O(1) X:
        fewer moduli as the correction shrinks (ozaki.correction_beta)."""
        return ozaki.correction_plan(bound, self.ws.n, self.gauss)

    def _hp_with(self, pl, ea, eb, out, **kw):
        pl = ozaki.fit_plan(pl, ea, eb)
        ozaki.gemm_residues(ea, eb, pl, self.res)
        ozaki.decode(self.res, ea, eb, pl, out, **kw)
        _counters["hp_calls"] += 1

    def entry(self, qhat):
        """Q = Q^ (3I - G) / 2 = Q^ - Q^ (G - I) / 2 (orthogonal.py:167-169)."""
        ws, hp, n = self.ws, self.hp, self.ws.n
        ea_qh = self._encode_q(qhat)                                     # Q^H (A role), Q^ (B role)
        self._hp(ea_qh, self.eb_q, ws.y, shift=-1.0, hermitian=True, pl=self.hq)  # G - I
        pc = self._correction_plan(ws.fro_norm(ws.y))
        ozaki.encode(qhat, n, n, "a", pc, out=self.ea_x)
        ozaki.encode(ws.y, n, n, "b", pc, out=self.eb_s)
        self._hp_with(pc, self.ea_x, self.eb_s, ws.q, alpha=-0.5, add=qhat)  # Q^ - Q^ (G - I) / 2

    def _encode_q(self, q):
        """Q as the B operand (self.eb_q) and Q^H as the A operand (returned):
        Gaussian planes — the same residues with the planes swapped; else one
        dual encode into self.ea_qh."""
        n = self.ws.n
        if self.gauss:
            ozaki.encode(q, n, n, "b", self.hq, out=self.eb_q)
            return ozaki.conj_view(self.eb_q)
        ozaki.encode_dual(q, n, n, self.hq, self.ea_qh, self.eb_q)
        return self.ea_qh

    def measure(self, a):
        ws, hp, n = self.ws, self.hp, self.ws.n
        ea_qh = self._encode_q(ws.q)                                    # Q^H (A role), Q (B role)
        if self.eb_a is None:
            self.eb_a = ozaki.encode(self.a, n, n, "b", self.hp_p)
        self._hp(ea_qh, self.eb_a, ws.p, pl=self.hp_p)                 # P = Q^H A
        ozaki.encode(ws.p, n, n, "a", self.hp_t, out=self.ea_x)
        self._hp(self.ea_x, self.eb_q, ws.that, pl=self.hp_t)          # T^ = P Q
        self._hp(ea_qh, self.eb_q, ws.y, shift=-1.0, hermitian=True, pl=self.hq)  # Y = Q^H Q - I

    def _lp_plans(self, norm_y, norm_w):
        return lp_plans(self.ws.n, norm_y, norm_w, self.gauss, self.lp)

    def update(self, restore_full_sigma, sigma_bound=None, norm_y=None, norm_w=None):
        ws, hp, lp, n = self.ws, self.hp, self.lp, self.ws.n
        if not restore_full_sigma:
            p_w2, p_xw = self._lp_plans(norm_y, norm_w)
            # a product below its own error budget is not formed (ozaki.lp_product_negligible):
            # W^2 only feeds the W^3 term of X W; X W itself is at most ||X|| ||W||
            skip_w2, skip_xw = lp_skips(norm_y, norm_w)
            if skip_xw:
                _sigma(ws, False, False, fused=True, drop_lp=True)       # S' = 2W - Y
            else:
                # two lp products instead of three: X W = YW - W^2 - W^3 with X = Y - W - W^2
                w_plan = None  # the plan self.lb holds W's encoding for
                if skip_w2:
                    pass
                elif self.gauss:
                    # W is exactly skew-Hermitian (sr_skew_c64): column j of W is -conj(row j),
                    # with the same scale, so W's B operand is its A operand with the
                    # Gaussian planes swapped and negated — one encoding of W, the
                    # sign folded into the decode (alpha = -1)
                    ozaki.encode(ws.w_lp, n, n, "a", p_w2, out=self.lb)       # W, A role
                    self._lp_with(p_w2, self.lb, ozaki.conj_view(self.lb), ws.w2, hermitian=True, alpha=-1.0)  # W^2
                    w_plan = p_w2
                else:
                    ozaki.encode(ws.w_lp, n, n, "b", p_w2, out=self.lb)       # W, B role
                    ozaki.encode(ws.w_lp, n, n, "a", p_w2, out=self.la)
                    self._lp_with(p_w2, self.la, self.lb, ws.w2, hermitian=self.w_skew)  # W^2 (W skew-Hermitian)
                    w_plan = p_w2
                _lib.call("sr_fused_lp_operand_c64", n, ws.y.re_ptr(), ws.y.im_ptr(), ws.y.ld, ws.w_lp.data_ptr(),
                          None if skip_w2 else ws.w2.data_ptr(), ws.w_lp.shape[1], ws.y_lp.data_ptr(), _stream())
                if p_xw is not w_plan:
                    ozaki.encode(ws.w_lp, n, n, "a" if self.gauss else "b", p_xw, out=self.lb)
                ozaki.encode(ws.y_lp, n, n, "a", p_xw, out=self.la)
                if self.gauss:
                    self._lp_with(p_xw, self.la, ozaki.conj_view(self.lb), ws.yw, alpha=-1.0)  # X W
                else:
                    self._lp_with(p_xw, self.la, self.lb, ws.yw)             # X W
                _sigma(ws, False, False, fused=True)                         # S' = S - 2I
        else:
            ozaki.encode(ws.w_lp, n, n, "b", lp, out=self.lb)            # W, B role (all lp products)
            ozaki.encode(ws.w_lp, n, n, "a", lp, out=self.la)
            self._lp(self.la, self.lb, ws.w2, hermitian=self.w_skew)     # W^2 (W skew-Hermitian)
            _downcast_y(ws)
            ozaki.encode(ws.w2, n, n, "a", lp, out=self.la)
            self._lp(self.la, self.lb, ws.w3, hermitian="skew" if self.w_skew else False)  # W^3
            ozaki.encode(ws.y_lp, n, n, "a", lp, out=self.la)
            self._lp(self.la, self.lb, ws.yw)                            # Y W
            ozaki.encode(ws.y_lp, n, n, "b", lp, out=self.lb)
            ozaki.encode(ws.w2, n, n, "a", lp, out=self.la)
            self._lp(self.la, self.lb, ws.w2y)                           # W^2 Y
            ozaki.encode(ws.w_lp, n, n, "b", lp, out=self.lb)
            ozaki.encode(ws.w2y, n, n, "a", lp, out=self.la)
            self._lp(self.la, self.lb, ws.w2yw)                          # W^2 Y W
            _sigma(ws, True, False)                                      # S' = S - 2I
        pc = hp if sigma_bound is None else self._correction_plan(sigma_bound)
        ozaki.encode(ws.q, n, n, "a", pc, out=self.ea_x)
        ozaki.encode(ws.sigma, n, n, "b", pc, out=self.eb_s)
        self._hp_with(pc, self.ea_x, self.eb_s, ws.q_next, alpha=0.5, add=ws.q)  # Q + Q S' / 2
        ws.q, ws.q_next = ws.q_next, ws.q


def lp_plans(n, norm_y, norm_w, gauss, default):
    """Plans for the fused update's W^2 and X W (X = Y - W - W^2) from
    ||Y||_F, ||W||_F: the products only enter S' multiplied by W (W^2,
    through X W) or as X W itself, so their allowed absolute error is the
    lp solve's own error in W (ozaki.lp_product_beta)."""
    if norm_y is None or norm_w is None or not (norm_w > 0.0):
        return default, default
    nx = norm_y + norm_w + norm_w * norm_w
    b_w2 = ozaki.lp_product_beta(norm_w * norm_w, n)      # W^2 error x ||W|| vs u ||W||
    b_xw = ozaki.lp_product_beta(nx, n)                   # (X W) error vs u ||W||
    return ozaki.plan(n, b_w2, b_w2, gauss), ozaki.plan(n, b_xw, b_xw, gauss)


def lp_skips(norm_y, norm_w):
    """(skip W^2, skip X W) for the fused update: the lp products that lie
    below their own error budget (ozaki.lp_product_negligible, the scales of
    lp_plans).  SR_LP_SKIP=0 forms every product (A/B runs)."""
    if norm_y is None or norm_w is None or not (norm_w > 0.0) or os.environ.get("SR_LP_SKIP") == "0":
        return False, False
    nx = norm_y + norm_w + norm_w * norm_w
    return ozaki.lp_product_negligible(norm_w * norm_w), ozaki.lp_product_negligible(nx)


def sigma_prime_bound(norm_y, norm_w, restore_full_sigma):
    """||S'||_F bound for S' = S - 2I = 2W - Y - YW + W^2 + W^3 (+ W^2 Y + W^2 Y W)
    from ||Y||_F and ||W||_F (sigma_merged_kernel, orthogonal.py:191-200)."""
    y, w = float(norm_y), float(norm_w)
    b = 2 * w + y + y * w + w * w + w ** 3
    if restore_full_sigma:
        b += w * w * y + w * w * y * w
    return b * (1 + 1e-6)


def make(kind, ws, a):
    if kind == "ozaki_std":
        return OzakiProducts(ws, a, gauss=False)
    if kind == "ozaki":
        return OzakiProducts(ws, a)
    if kind == "dmma":
        return DmmaProducts(ws, a)
    raise ValueError("unknown gemm kind %r" % (kind,))


def ensure_full_sigma_buffers(ws):
    if ws.w2y is None:
        ws.w2y = lp_empty(ws.n, device=ws.w_lp.device)
        ws.w2yw = lp_empty(ws.n, device=ws.w_lp.device)


__all__ = ["DmmaProducts", "OzakiProducts", "make", "ensure_full_sigma_buffers", "ZPlanar"]
