"""ddschur.dd: scalar EFTs are host utilities — the reference's own."""
from . import reference_module

U_HP = 2.0 ** -106


def __getattr__(name):
    if name.startswith("__"):
        raise AttributeError(name)
    return getattr(reference_module("dd"), name)
