"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This package generates geometry (points, outward normals, panel weights) and
densities with the shapes and distributions of BASELINE.json's configs.  It holds
none of the method's arithmetic (no kernels, no tree, no translations) so that it
can serve both sides of the parity check.
"""
