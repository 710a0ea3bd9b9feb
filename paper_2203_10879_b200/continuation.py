"""Parameter-continuation driver (BASELINE config 5): refine A(t_j) = A0 + t_j A1
for t_0 < t_1 < ..., starting each refinement from the refined Q of the
previous parameter value (the reference's de-facto resume is to feed
`pair.q` back into `refine_template`).  Every step is a full
`refine_template` call; A(t_j) is formed on the device."""
import torch

from .matrix import ZPlanar
from .refine import RefineConfig, refine_template


def refine_continuation(a0, a1, ts, qhat0, cfg=None, device=None):
    """Returns [(t_j, SchurPair, RefineReport)] for every t_j in ts."""
    cfg = RefineConfig(precision="fp64") if cfg is None else cfg
    device = torch.device("cuda") if device is None else torch.device(device)
    a0 = ZPlanar.from_any(a0, device=device, force_complex=True)
    a1 = ZPlanar.from_any(a1, device=device, force_complex=True)
    at = ZPlanar.empty(a0.rows, device=device)
    q = qhat0
    out = []
    for t in ts:
        torch.add(a0.re_buf, a1.re_buf, alpha=float(t), out=at.re_buf)
        torch.add(a0.im_buf, a1.im_buf, alpha=float(t), out=at.im_buf)
        pair, rep = refine_template(at, q, cfg, device=device)
        out.append((float(t), pair, rep))
        q = pair.q
    return out
