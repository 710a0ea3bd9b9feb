"""GPU solve of stril(T L - L T) = -E, reference-shaped API.

  TriEqProblem / TriEqSolution  /root/reference/pkg/src/ddschur/trisolve.py:58-84
  solve_block                   trisolve.py:243-262
  solve_scalar                  trisolve.py:148-161
  stats / reset_stats           trisolve.py:36-47
  SeparationError / NonFiniteError trisolve.py:50-55

The kernel (csrc/trisolve.cu) is a blocked anti-diagonal wavefront; n_min
is accepted for signature compatibility and does not change the result
beyond rounding (L is unique).  solve_scalar (the reference's
entrywise substitution, Algorithm 2) is the same unique L, so it runs the
same kernel; the two differ only in the invocation counters, which follow
the reference's accounting (one Sylvester solve per split of the halving
recursion at n_min).  The arithmetic follows the operands: complex128
(the reference's binary64 lp, numpy's default) or complex64 (FP64 mode);
numpy in, numpy out.
"""
import dataclasses

import numpy as np
import torch

from . import _lib
from .errors import NonFiniteError, SeparationError
from .matrix import even

DEFAULT_NMIN = 4

_stats = {"scalar_solves": 0, "block_solves": 0, "sylvester_solves": 0}


def reset_stats():
    """Zero the solver invocation counters (trisolve.py:36-40)."""
    for key in _stats:
        _stats[key] = 0


def stats():
    """A copy of the solver invocation counters (trisolve.py:43-47)."""
    return dict(_stats)


def _sylvester_count(n, n_min):
    """Splits of _block_solve's halving recursion (trisolve.py:223-240)."""
    if n <= n_min:
        return 0
    n1 = n // 2
    return 1 + _sylvester_count(n1, n_min) + _sylvester_count(n - n1, n_min)


@dataclasses.dataclass
class TriEqProblem:
    t: object
    e: object
    clip_threshold: float | None = None


@dataclasses.dataclass
class TriEqSolution:
    l: object
    clipped_count: int


class SolverWorkspace:
    """Device scratch for repeated solves at one size (no per-call allocation)."""

    def __init__(self, n, lp_dtype=torch.complex64, device="cuda"):
        self.n = n
        self.lp_dtype = lp_dtype
        c64 = 1 if lp_dtype == torch.complex64 else 0
        nbytes = _lib.load().sr_trisolve_workspace_bytes(n, c64)
        self.ws = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
        self.clipped = torch.zeros(1, dtype=torch.int64, device=device)
        self.flags = torch.zeros(1, dtype=torch.int32, device=device)


def solve_lp_device(t, e, l, n, clip_threshold, work, stream):
    """Launch the solver on (n, ld) interleaved lp tensors; counters and
    flags accumulate into work.clipped / work.flags (read by the caller)."""
    clip = 0.0 if clip_threshold is None else float(clip_threshold)
    name = "sr_trisolve_c64" if t.dtype == torch.complex64 else "sr_trisolve_c128"
    _lib.call(name, n, t.data_ptr(), e.data_ptr(), t.shape[1], l.data_ptr(), clip, work.clipped.data_ptr(),
              work.flags.data_ptr(), work.ws.data_ptr(), work.ws.numel(), stream)


def _solve(problem, lp_dtype, device):
    is_np = not torch.is_tensor(problem.t)
    t = torch.as_tensor(np.asarray(problem.t) if is_np else problem.t)
    e = torch.as_tensor(np.asarray(problem.e) if not torch.is_tensor(problem.e) else problem.e)
    if t.dim() != 2 or t.shape[0] != t.shape[1]:
        raise ValueError("t must be square")
    if e.shape != t.shape:
        raise ValueError("e must match the shape of t")
    clip = problem.clip_threshold
    if clip is not None and not clip > 0:
        raise ValueError("clip_threshold must be positive")
    if lp_dtype is None:  # the operands' precision (the reference coerces to complex128)
        lp_dtype = torch.complex64 if t.dtype == torch.complex64 else torch.complex128
    n = t.shape[0]
    ld = even(max(n, 1))
    td = torch.zeros((n, ld), dtype=lp_dtype, device=device)
    ed = torch.zeros((n, ld), dtype=lp_dtype, device=device)
    td[:, :n] = t.to(device=device, dtype=lp_dtype)
    ed[:, :n] = e.to(device=device, dtype=lp_dtype)
    if bool(torch.any(torch.tril(td[:, :n], -1) != 0)):
        raise ValueError("t must be upper triangular with exact zeros below")
    if bool(torch.any(torch.triu(ed[:, :n]) != 0)):
        raise ValueError("e must be strictly lower triangular")
    l = torch.empty((n, ld), dtype=lp_dtype, device=device)
    work = SolverWorkspace(n, lp_dtype, device)
    solve_lp_device(td, ed, l, n, clip, work, torch.cuda.current_stream().cuda_stream)
    flags = int(work.flags.item())
    if flags & _lib.SR_FLAG_SEPARATION:
        raise SeparationError("diagonal separation is exactly zero")
    lv = l[:, :n]
    if not bool(torch.isfinite(torch.view_as_real(lv)).all()):
        raise NonFiniteError("solution contains non-finite entries")
    out = lv.cpu().numpy() if is_np else lv
    return TriEqSolution(l=out, clipped_count=int(work.clipped.item()))


def solve_block(problem, n_min=DEFAULT_NMIN, lp_dtype=None, device="cuda"):
    """solve_block(TriEqProblem) -> TriEqSolution on the GPU (trisolve.py:243-262).

    Validates like trisolve.py:87-101, raises SeparationError on an exactly
    repeated diagonal and NonFiniteError on overflow, like the reference."""
    if n_min < 2:
        raise ValueError("n_min must be at least 2")
    sol = _solve(problem, lp_dtype, device)
    _stats["block_solves"] += 1
    _stats["sylvester_solves"] += _sylvester_count(np.shape(problem.t)[0], n_min)
    return sol


def solve_scalar(problem, lp_dtype=None, device="cuda"):
    """solve_scalar(TriEqProblem) -> TriEqSolution (trisolve.py:148-161): the
    same unique L as solve_block, with the reference's error behaviour."""
    sol = _solve(problem, lp_dtype, device)
    _stats["scalar_solves"] += 1
    return sol
