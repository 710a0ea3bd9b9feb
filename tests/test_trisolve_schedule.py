"""CPU check of the lp solver's update schedule (csrc/trisolve.cu).

The wavefront solves tile (I, M) of L (I >= M, N x N tiles of 32) on level
(N-1-I) + M.  Its right-hand side needs every column term T_IK L_KM (K > I)
and row term L_IJ T_JM (J < M).  The kernels split these contributions into
the SOLVE fold (sources on the previous level), the NEAR band and the FAR
batches.  This test replays the host loop's index sets for several N and
checks that every (source, target) pair is applied exactly once, after the
source tile is solved and no later than the launch that solves the target —
the invariant the parity tests rely on.  Mirrors solve<C>() and the kernels'
tile enumeration line by line (BW = 4; FAR_LA = 1 as compiled, 2 and 3 to keep
the index algebra general)."""
import collections

import pytest

BW = 4


def level(N, I, M):
    return (N - 1 - I) + M


def schedule(N, FAR_LA):
    """-> {(target, source, kind): time} with time = (lev, phase): phase 0 = SOLVE
    fold of launch lev, 1 = NEAR of lev, 2 = FAR issued after SOLVE(lev)
    (needed by level >= its first target level)."""
    applied = collections.Counter()
    when = {}

    def add(tgt, src, kind, t):
        applied[(tgt, src, kind)] += 1
        when[(tgt, src, kind)] = t

    for lev in range(N):
        # SOLVE(lev): tiles (M + N - 1 - lev, M), M in [0, lev]; fold level lev-1 sources
        for M in range(lev + 1):
            I = M + N - 1 - lev
            if lev >= 1 and M <= lev - 1:
                add((I, M), (M + N - lev, M), "col", (lev, 0))
            if lev >= 1 and I >= N - lev:
                add((I, M), (I, I - N + lev), "row", (lev, 0))
        # NEAR(lev): sources on level lev-1 into levels lev+1 .. lmax
        if lev >= 1:
            b = (lev - 1) // BW
            lmax = min(N - 1, BW * (b + 1 + FAR_LA) - 1)
            for lv in range(lev + 1, lmax + 1):
                for M in range(lv + 1):
                    I = M + N - 1 - lv
                    if M <= lev - 1:
                        add((I, M), (M + N - lev, M), "col", (lev, 1))
                    if I >= N - lev:
                        add((I, M), (I, I - N + lev), "row", (lev, 1))
        # FAR(b) after SOLVE(4b+3)
        if lev % BW == BW - 1:
            b = lev // BW
            first_level = BW * (b + 1 + FAR_LA)
            h = N - first_level
            if h >= 1:
                for M in range(min(BW * b + BW, N)):            # COL lines
                    for t in range(h):
                        I = M + t
                        for k in range(BW):
                            K = M + N - BW * b - BW + k
                            if K <= N - 1:
                                add((I, M), (K, M), "col", (lev, 2))
                for I in range(N - BW - BW * b, N):            # ROW lines
                    for t in range(h):
                        M = I - N + 1 + first_level + t
                        for k in range(BW):
                            J = I - N + 1 + BW * b + k
                            if J >= 0:
                                add((I, M), (I, J), "row", (lev, 2))
    return applied, when


@pytest.mark.parametrize("FAR_LA", [1, 2, 3])
@pytest.mark.parametrize("N", [1, 2, 3, 5, 8, 9, 12, 13, 16, 17, 21, 33, 40])
def test_every_contribution_applied_once_in_order(N, FAR_LA):
    applied, when = schedule(N, FAR_LA)
    need = set()
    for I in range(N):
        for M in range(I + 1):
            for K in range(I + 1, N):
                need.add(((I, M), (K, M), "col"))
            for J in range(M):
                need.add(((I, M), (I, J), "row"))
    assert set(applied) == need
    assert all(c == 1 for c in applied.values())
    for (tgt, src, kind), (lev, phase) in when.items():
        ls, lt = level(N, *src), level(N, *tgt)
        assert ls < lt
        if phase == 0:      # SOLVE fold: source solved by the previous launch
            assert lev == lt and ls == lev - 1
        elif phase == 1:    # NEAR(lev) runs after SOLVE(lev-1), before SOLVE(lev+1)
            assert ls == lev - 1 and lt >= lev + 1
        else:               # FAR(b) after SOLVE(4b+3); SOLVE(l) waits FAR(l/4 - 1 - FAR_LA)
            b = lev // BW
            assert BW * b <= ls <= lev
            assert lt >= BW * (b + 1 + FAR_LA)
            assert (lt // BW) - 1 - FAR_LA >= b   # the wait at level 4*(lt//4) covers FAR(b)
