"""ddschur.orthogonal: Newton-Schulz / merged update on the GPU; qr_retract
(not on the default path) from the reference."""
from paper_2203_10879_b200.errors import NormTooLarge  # noqa: F401
from paper_2203_10879_b200.orthogonal import merged_update, newton_schulz_step  # noqa: F401
from paper_2203_10879_b200.refine import OrthoStrategy  # noqa: F401

from . import reference_module


def qr_retract(m):
    return reference_module("orthogonal").qr_retract(m)


def __getattr__(name):
    if name.startswith("__"):
        raise AttributeError(name)
    return getattr(reference_module("orthogonal"), name)
