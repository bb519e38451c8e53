"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A numpy (+ one small C file) restatement of the reference's per-step
pipeline, ``clothsim.Simulation.step`` (reference
``pkg/src/clothsim/stepper.py:454-624``) and every stage it calls.  Each
function cites the reference file:line it follows.

Rules:
  * Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
    ``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
    product (``paper_2403_19272_b200``) never imports it and has no CPU
    fallback.
  * Parity is PINNED: ``tests/golden/make_golden.py`` runs the real reference
    (importable in the build container from /root/reference) and commits its
    outputs under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this
    oracle reproduces them bit-for-bit (pair sets, row order, CCD hit sets,
    TOIs, solver outputs and multi-step trajectories).
  * Scene setup (mesh topology, H, eigenbasis) is shared input taken from the
    product's host setup modules, which are themselves pinned against the
    reference's arrays in ``tests/test_setup_parity.py``.

Arithmetic follows numpy's evaluation order exactly (einsum over 3 terms =
(a0 b0 + a2 b2) + a1 b1, sequential norms, OpenBLAS's forward FMA chain for
the 4x4 cubic fit - restated in ``oracle/c/ccd_fit.c`` so the oracle does not
depend on the host's BLAS kernel).
"""
