"""Alias of the reference's ssimkit.color onto the B200 engine (see __init__.py)."""
from . import lookup


def __getattr__(name):
    return lookup("color", name)
