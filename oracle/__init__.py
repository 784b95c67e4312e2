"""CPU ORACLE for the immersed Newmark IMEX spectral cell method (arXiv 2310.14712).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or run
anything under ``oracle/``.  The product path (``paper_2310_14712_b200``)
never imports it and fails loudly when its CUDA library is missing.

Plain, slow, obviously-correct fp64 numpy/scipy code that follows the paper
step by step; it shares no code, headers, tables or constant generators with
the CUDA path.  Each function cites the PAPER.md passage (``P:line``) it
follows; readings of silent/garbled passages are the C-numbers of DESIGN.md §3.

Modules
-------
basis        GLL / Gauss-Legendre rules, Lagrange basis
geometry     void membership, lattice cut test, spacetree, cell classes
             (readings C6, C7, C17)
elements     uncut / cut element matrices (C5)
assembly     DOF map, partition, global sparse M and K or element-by-element
             operator, point-source f_x
integrators  CDM, trapezoidal Newmark, Newmark IMEX (C1-C4)
spectra      critical time steps and the Fig. 2 study
run          config dict -> system -> IMEX run

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` (see DESIGN.md §4 for the pin list); none is
"parity unpinned".
"""
