"""B200-native GACER multi-tenant executor (arXiv 2304.11745).

The product is ``libgacer.so`` (C ABI, include/gacer.h) built from
``csrc/``; ``gacer`` is the thin ctypes binding and ``runtime`` the
torch-plumbing helpers (device buffers, layouts) used by tests and bench.
"""
from . import gacer  # noqa: F401
