"""B200-native IFGF matvec (arXiv 2010.02857): C-ABI library libifgf.so + thin binding.

``inputs`` (seeded synthetic workloads) imports without the CUDA library;
``Plan``, ``direct``, ``partition`` and ``bench_dfma`` load ``libifgf.so``
on first use and raise if it is missing (no CPU fallback).
"""
from . import inputs  # noqa: F401

_LAZY = ("Plan", "direct", "partition", "bench_dfma", "version", "IfgfError")


def __getattr__(name):
    if name in _LAZY:
        from . import ifgf as _m
        return getattr(_m, name)
    raise AttributeError(name)
