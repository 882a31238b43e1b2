"""CPU fp64 ORACLE for the batched IPC + ABD Newton step of Taccel (arXiv 2504.12908).

*** TEST INFRASTRUCTURE ONLY. ***  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu-baseline / ``--impl reference`` leg may import anything under ``oracle/``.  The product path
(``paper_2504_12908_b200``'s CUDA library and its binding) never imports, links or executes it,
and the oracle never imports the product path: the two share only the seeded input generator
``paper_2504_12908_b200.scenes`` (geometry and scripted targets, none of the method's arithmetic).

What it is: a plain, slow, single-threaded, obviously-correct implementation of what one time
step computes, written in numpy / plain PyTorch CPU ops in float64:

  mesh.py      rest quantities, lumped masses, surfaces, rest areas, reduced mass M^y
  distance.py  point-triangle / edge-edge closest-point type and squared distance
  energy.py    incremental potential terms (inertia, Neo-Hookean, orthogonality, gravity,
               log barrier, augmented Lagrangian); gradients and Hessians are obtained by
               automatic differentiation (torch.func) of the plain energy definitions, and
               PSD projections by numpy.linalg.eigh (library primitives)
  contact.py   brute-force candidate / active sets and additive CCD
  solver.py    projected Newton with an exact sparse direct solve (or block-Jacobi PCG),
               ACCD-bounded backtracking line search, AL outer loop, velocity update
  readout.py   gel-surface deformation and marker flow

Paper readings (garbled / silent passages) are the ones listed in DESIGN.md §3; each function
cites the passage it follows.  Pins (tests that tie the oracle to something other than itself)
live in tests/test_oracle_*.py.  Parity status: every function is pinned except where its
docstring says "parity unpinned".
"""
