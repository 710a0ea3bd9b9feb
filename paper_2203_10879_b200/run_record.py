"""JSON run record, schema v1: the reference's report
format (/root/reference/pkg/src/ddschur/cli.py:30-144) — one JSON object per
refinement with the input spec, the configuration, the RefineReport and the
verify_pair residuals, plus an optional bench block.  Non-finite floats
serialise as null.  (The command-line front end itself is out of scope.)"""
import json
import math

from .refine import OrthoStrategy, RefineStatus

SCHEMA_VERSION = 1
SPEC_KINDS = ("randn", "randn-real", "wilkinson", "clustered", "file")  # generators.MatrixKind values
SPEC_KEYS = ("kind", "n", "seed", "cluster_count", "cluster_size", "cluster_radius", "cond_x", "path")
CONFIG_KEYS = ("tol_factor", "max_iters", "n_min", "clip_threshold", "ortho", "skip_final_ortho", "seed",
               "restore_full_sigma")
REPORT_KEYS = ("iterations", "residual_history", "hp_matmul_count", "clipped_total", "status", "wall_time",
               "skip_fired", "detail")
RESIDUAL_KEYS = ("ortho_residual", "tri_residual", "similarity_residual")
BENCH_KEYS = ("hp_seconds", "lp_seconds", "hp_fraction")


def _num(x):
    x = float(x)
    return x if math.isfinite(x) else None


def make_spec(kind, n, seed=0, cluster_count=0, cluster_size=0, cluster_radius=0.0, cond_x=1.0, path=None):
    """The input-matrix spec block (generators.MatrixSpec.to_dict fields)."""
    if kind not in SPEC_KINDS:
        raise ValueError("unknown matrix kind %r" % (kind,))
    return dict(kind=kind, n=int(n), seed=int(seed), cluster_count=int(cluster_count),
                cluster_size=int(cluster_size), cluster_radius=float(cluster_radius), cond_x=float(cond_x),
                path=path)


def config_to_dict(cfg):
    return {k: (cfg.ortho.value if k == "ortho" else getattr(cfg, k)) for k in CONFIG_KEYS}


def report_to_dict(rep):
    return dict(iterations=rep.iterations,
                residual_history=[[_num(e), _num(y)] for e, y in rep.residual_history],
                hp_matmul_count=rep.hp_matmul_count, clipped_total=rep.clipped_total, status=rep.status.value,
                wall_time=rep.wall_time, skip_fired=rep.skip_fired, detail=rep.detail)


def residuals_to_dict(res):
    return {k: _num(getattr(res, k)) for k in RESIDUAL_KEYS}


def build_run_record(spec, cfg, report, residuals, bench=None):
    rec = dict(schema=SCHEMA_VERSION, spec=dict(spec), config=config_to_dict(cfg), report=report_to_dict(report),
               residuals=residuals_to_dict(residuals))
    if bench is not None:
        rec["bench"] = dict(bench)
    return rec


def _expect(cond, msg):
    if not cond:
        raise ValueError("invalid run record: %s" % msg)


def validate_run_record(rec):
    """Check a record against schema v1; returns it unchanged."""
    _expect(isinstance(rec, dict), "not an object")
    extra = set(rec) - {"schema", "spec", "config", "report", "residuals", "bench"}
    _expect(not extra, "unknown keys %s" % sorted(extra))
    _expect(rec.get("schema") == SCHEMA_VERSION, "schema must be %d" % SCHEMA_VERSION)
    spec = rec.get("spec")
    _expect(isinstance(spec, dict) and set(spec) == set(SPEC_KEYS), "bad spec keys")
    _expect(spec["kind"] in SPEC_KINDS, "bad spec kind")
    cfg = rec.get("config")
    _expect(isinstance(cfg, dict) and set(cfg) == set(CONFIG_KEYS), "bad config keys")
    _expect(cfg["ortho"] in {s.value for s in OrthoStrategy}, "bad ortho")
    rep = rec.get("report")
    _expect(isinstance(rep, dict) and set(rep) == set(REPORT_KEYS), "bad report keys")
    _expect(rep["status"] in {s.value for s in RefineStatus}, "bad status %r" % (rep["status"],))
    hist = rep["residual_history"]
    _expect(isinstance(hist, list) and all(isinstance(r, list) and len(r) == 2 for r in hist),
            "residual_history must be a list of pairs")
    _expect(len(hist) == rep["iterations"] + 1, "residual_history must have iterations + 1 rows")
    res = rec.get("residuals")
    _expect(isinstance(res, dict) and set(res) == set(RESIDUAL_KEYS), "bad residual keys")
    if "bench" in rec:
        _expect(isinstance(rec["bench"], dict) and set(rec["bench"]) == set(BENCH_KEYS), "bad bench keys")
    return rec


def dumps(rec):
    """Compact JSON text of a validated record."""
    return json.dumps(validate_run_record(rec), sort_keys=True)


__all__ = ["SCHEMA_VERSION", "make_spec", "config_to_dict", "report_to_dict", "residuals_to_dict",
           "build_run_record", "validate_run_record", "dumps"]
