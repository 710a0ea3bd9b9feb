"""CPU-side checks of the drop-in boundary: libsr.so loads and exports every
symbol include/sr.h declares; host-side API validation mirrors the
reference (RefineConfig checks, refine.py:72-82)."""
import os
import re

import pytest

from paper_2203_10879_b200 import RefineConfig, _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(REPO, "include", "sr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*|unsigned long long)\s+(sr_\w+)\s*\(", src, re.M)))


def test_header_and_binding_agree():
    assert set(declared_symbols()) == set(_lib.SIGNATURES)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.sr_version() >= 1
    assert lib.sr_reduce_workspace_bytes() > 0
    assert lib.sr_trisolve_workspace_bytes(8192, 1) > 0


def test_invalid_arguments_are_rejected_without_a_gpu():
    lib = _lib.load()
    # negative sizes and odd leading dimensions are argument errors
    assert lib.sr_zgemm_f64(0, -1, 4, 4, 1.0, 0.0, 16, 16, 4, 16, 16, 4, 16, 16, 4, None) == _lib.SR_EINVAL
    assert lib.sr_zgemm_f64(0, 4, 4, 4, 1.0, 0.0, 16, 16, 3, 16, 16, 4, 16, 16, 4, None) == _lib.SR_EINVAL
    assert lib.sr_cgemm_c64(1, 4, 4, 4, 16, 4, 16, 4, 16, 4, None) == _lib.SR_EINVAL
    with pytest.raises(ValueError):
        _lib.check(_lib.SR_EINVAL, "probe")


def test_refine_config_validation():
    with pytest.raises(ValueError):
        RefineConfig(tol_factor=0.0)
    with pytest.raises(ValueError):
        RefineConfig(max_iters=0)
    with pytest.raises(ValueError):
        RefineConfig(n_min=1)
    with pytest.raises(ValueError):
        RefineConfig(clip_threshold=-1.0)
    with pytest.raises(ValueError):
        RefineConfig(precision="fp32")
    assert RefineConfig().precision == "dd"


def test_correction_beta_tracks_the_correction_size():
    """Operand precision of the correction products (Q + Q S'/2): full hp for
    an O(1) correction, fewer bits (fewer moduli) as ||S'|| shrinks, never below
    the lp precision; a non-finite bound falls back to full hp."""
    from paper_2203_10879_b200 import ozaki
    n = 8192
    assert ozaki.correction_beta(1.0, n) == ozaki.HP_BETA
    assert ozaki.correction_beta(1e-6, n) == 53 + 3 - 19 + 7
    # S needs log2(n)/2 fewer bits than X (its truncation is not amplified by the row length)
    assert ozaki.correction_beta(1e-6, n, operand="s") == 53 + 3 - 19
    pl = ozaki.correction_plan(1e-6, n)
    assert (pl.beta_a, pl.beta_b) == (53 + 3 - 19 + 7, 53 + 3 - 19)
    assert pl.nmod <= ozaki.plan(n, pl.beta_a, pl.beta_a).nmod
    assert ozaki.correction_beta(1e-30, n) == ozaki.LP_BETA
    assert ozaki.correction_beta(0.0, n) == ozaki.LP_BETA
    assert ozaki.correction_beta(float("nan"), n) == ozaki.HP_BETA
    assert ozaki.correction_beta(float("inf"), n) == ozaki.HP_BETA
    betas = [ozaki.correction_beta(10.0 ** -k, n) for k in range(0, 20)]
    assert betas == sorted(betas, reverse=True)
    mods = [ozaki.plan(n, b, b).nmod for b in betas]
    assert mods[0] == ozaki.plan(n, ozaki.HP_BETA, ozaki.HP_BETA).nmod and mods[-1] < mods[0]


def test_ddschur_import_shim_maps_the_hot_path():
    """tools/ddschur_shim: `import ddschur` resolves the hot-path names to the
    B200 drop-in (the reference's own tests can then run against it on a
    machine with a GPU and the reference source, tools/run_reference_tests.sh)."""
    import subprocess
    import sys
    code = ("import ddschur, paper_2203_10879_b200 as p; "
            "from ddschur.ddmatrix import DDMatrix, frobenius_norm, stril_extract; "
            "from ddschur.trisolve import solve_block, solve_scalar, stats, reset_stats; "
            "from ddschur.orthogonal import newton_schulz_step, merged_update; "
            "from ddschur.refine import RefineConfig; "
            "assert DDMatrix is p.DDMatrix and solve_scalar is p.solve_scalar and stats is p.stats; "
            "assert newton_schulz_step is p.newton_schulz_step and RefineConfig().precision == 'dd'; "
            "print('ok')")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(REPO, "tools", "ddschur_shim"), REPO]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr


def test_negligible_lp_products_rule(monkeypatch):
    """The fused update leaves out an lp product only when its norm bound is
    below the error the adaptive plans allow it (2^-26 ||W||_F): W^2 (which
    only feeds the W^3 term) from ||W||_F^2 <= 2^-26, X W from ||X||_F <= 2^-26."""
    from paper_2203_10879_b200 import ozaki, products

    assert ozaki.lp_product_negligible(2.0 ** -26) and not ozaki.lp_product_negligible(2.0 ** -25.9)
    assert not ozaki.lp_product_negligible(float("nan")) and not ozaki.lp_product_negligible(float("inf"))
    monkeypatch.delenv("SR_LP_SKIP", raising=False)
    assert products.lp_skips(None, 1e-9) == (False, False)           # no norms (merged_update export): every product
    assert products.lp_skips(1e-7, 0.0) == (False, False)
    assert products.lp_skips(1e-7, 1e-3) == (False, False)           # first updates: W^2 matters
    assert products.lp_skips(1e-10, 1e-5) == (True, False)           # ||W||^2 = 1e-10 < 2^-26, ||X|| ~ 1e-5 is not
    assert products.lp_skips(1e-13, 2e-9) == (True, True)            # last update of a converging run
    assert products.lp_skips(1e-6, 2e-9) == (True, False)            # a large orthogonality defect keeps X W
    monkeypatch.setenv("SR_LP_SKIP", "0")
    assert products.lp_skips(1e-13, 2e-9) == (False, False)
