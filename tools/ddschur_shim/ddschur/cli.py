"""ddschur.cli: outside the hot path — the unmodified reference module."""
from . import reference_module


def __getattr__(name):
    if name.startswith("__"):
        raise AttributeError(name)
    return getattr(reference_module("cli"), name)
