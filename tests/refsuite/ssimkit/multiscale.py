"""Alias of the reference's ssimkit.multiscale onto the B200 engine (see __init__.py)."""
from . import lookup


def __getattr__(name):
    return lookup("multiscale", name)
