"""Float64 CPU oracle for the MS-LLR data-consistency operator (arxiv 2310.05647).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2310_05647_b200`` + ``libmrfnufft.so``) never imports, calls or links it, and the
oracle shares no code, header, table or constant generator with the CUDA path.

Layers:
  (i)  ``oracle.nufft.nudft_*``  -- the plain definition (direct non-uniform DFT) of
       A = F_u C (Eq. (1) ``data_ac``) and of its adjoint A* (PAPER.md:221).
  (ii) ``oracle.nufft.grid_*``   -- the Kaiser-Bessel gridding NUFFT the GPU reproduces, step by
       step in the order of SURVEY.md §8(c)(ii) (deapodize -> pad -> FFT -> interpolate, and the
       exact transpose), written out with numpy/scipy primitives and no blocking or fusion.
  (iii) ``oracle.cg``             -- CG on (A^H A + mu I) x = A^H y + mu z with global inner
       products (BASELINE.json north_star; not in the paper, which takes gradient steps with
       A*(A X - b), Eq. (15)).

Every function cites the passage it follows.  Pins (``tests/test_oracle_*.py``, ``-m "not gpu"``)
tie each function to something other than itself: brute-force NUDFT, ``numpy.fft`` on a
Cartesian trajectory, closed forms (delta image, single DC sample, KB Fourier transform by
quadrature), the adjoint identity, Hermitian/PSD structure, A^H A = I on a full Cartesian
trajectory, and CG = Krylov projection / dense solve.
"""
from . import kb, nufft, cg, pcg, match, dcf, llr, manifold, msllr  # noqa: F401
