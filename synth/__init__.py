"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no kernel, no FFT, no gridding): only the
trajectories, images, coil maps and noise draws that both sides consume.  See
``synth.inputs`` and DESIGN.md §"Input recipe".
"""
from .inputs import *  # noqa: F401,F403
