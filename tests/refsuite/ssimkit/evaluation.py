"""Alias of the reference's ssimkit.evaluation: outside the engine's scope (see __init__.py)."""
from . import lookup


def __getattr__(name):
    return lookup("evaluation", name)
