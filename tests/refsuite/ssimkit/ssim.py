"""Alias of the reference's ssimkit.ssim onto the B200 engine (see __init__.py)."""
from . import lookup


def __getattr__(name):
    return lookup("ssim", name)
