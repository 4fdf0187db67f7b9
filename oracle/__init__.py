"""CPU ORACLE — test infrastructure only.

This package is a plain-numpy restatement of the reference ``paracycle``
algorithm for the PTL-cycled parabolic-operator path (SPEC.md:84-400,
PAPER.md Eq. 2-5 and Appendix A, mesh.py conventions), extended to the
spherical (r, theta, phi) geometry that BASELINE.json's north star asks for.

It exists ONLY as the checker: ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it.
The product package ``paper_2403_01004_b200`` never imports it, and the
product path fails loudly when its CUDA library is missing.

Parity pinning:
  * Cartesian metric mode is pinned to the SPEC's known-answer examples and to
    the reference ``mesh.py`` (dual volumes, ghost rules), see
    ``tests/golden/`` and ``tests/test_oracle_kat.py``.
  * The spherical metric, the axis (pole) treatment, the vector-viscosity
    metric terms and the 19-point aligned-conduction stencil are NEW design
     with no reference code or test: for those the oracle is
    "parity unpinned" against the reference and is checked by property tests
    (conservation, symmetry, negative semi-definiteness, 1-D reductions).

Every array operation is written in an explicit order (no implicit
reassociation, no fused multiply-add) so that the CUDA kernels, compiled with
``-fmad=false`` and the same operation order, reproduce it bit for bit.
"""
