"""ddschur.refine on the B200 drop-in (dd mode, host DDMatrix results)."""
import dataclasses

from paper_2203_10879_b200 import refine as _r
from paper_2203_10879_b200.refine import (NotSymmetric, OrthoStrategy, RefineReport, RefineStatus,  # noqa: F401
                                          VerifyResiduals, verify_pair)

RefineConfig = _r.RefineConfig  # default precision "dd": the reference's pair


def _host(pair):
    for k in ("q", "t"):
        v = getattr(pair, k)
        if hasattr(v, "to_ddmatrix"):
            setattr(pair, k, v.to_ddmatrix())
    return pair


def refine_template(a, qhat, cfg=None):
    pair, rep = _r.refine_template(a, qhat, cfg)
    return _host(pair), rep


def refine_mixed(a, cfg=None):
    from paper_2203_10879_b200 import refine_mixed as _m
    pair, rep = _m(a, cfg)
    return _host(pair), rep


def refine_symmetric(a, cfg=None):
    from paper_2203_10879_b200 import refine_symmetric as _s
    pair, rep = _s(a, cfg)
    return _host(pair), rep


__all__ = ["RefineConfig", "RefineReport", "RefineStatus", "NotSymmetric", "OrthoStrategy", "VerifyResiduals",
           "refine_template", "refine_mixed", "refine_symmetric", "verify_pair", "dataclasses"]
