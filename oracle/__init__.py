"""AIMx fp64 CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import anything under
``oracle/``.  The product path (``paper_2009_02281_b200``) never imports,
links or executes it, and this package never imports the product path: the
two share no code; only ``aimx_inputs`` (seeded meshes and vectors, no method
arithmetic) serves both.

Plain, slow, obviously correct NumPy/SciPy code in float64/complex128 that
follows arxiv 2009.02281 (PAPER.md, cited as ``P:<line>`` with the LaTeX
label) step by step:

* ``kernels``       G, G_s, G_d (eq:hgf P:172, eq:hgfs P:226, eq:hgfd P:230)
* ``mesh``          RWG basis
* ``grid``          AIM grid, stencils, near-region map
* ``projection``    moment-matched projection weights P^(A), P^(phi) (P:109-110,
                    P:198)
* ``static_near``   L_s,NR by direct integration with G_s (eq:Lmatdecomp2 P:267,
                    change (a) P:297)
* ``precorrection`` L_s,P = W H_s,NR P (eq:aimLPs P:276, eq:Hsmm P:321)
* ``convolution``   3-level Toeplitz H(k0) applied by zero-padded FFT
                    (eq:Hmn P:305, eq:Hmm P:335)
* ``aimx``          the AIMx EFIE matvec (eq:LAIMx P:283, eq:EFIEAIMx P:288)
* ``direct``        dense direct-integration MoM (the paper's "direct" mode),
                    optionally with k0^2 G_lin integrated analytically
* ``linear_term``   the linear-term modification: G_lin = -r/(8 pi),
                    C_lin = L_lin - W H_lin P on overlapping pairs
                    (eq:linterm P:363, eq:Lmatdecomplin P:386)
* ``gmres``         restarted GMRES with the static diagonal preconditioner
* ``kop``           AIMx for the double-layer operator K (eq:opK P:408,
                    eq:KAIMx P:457; NEXT #1)
* ``aim``           the conventional AIM (per-frequency near region and
                    precorrection, eq:aimL P:190, eq:aimLP P:205)

Every reading of a silent/ambiguous/garbled passage is listed in DESIGN.md
("Readings") with the AMB-n tag used in comments here.

Parity status: every function is pinned by a ``-m "not gpu"`` test in
``tests/test_oracle_*.py`` against closed forms, brute force, invariants or
the paper's printed values.  The sign of ``kop``'s residue term (reading R24)
and the PMCHWT composition and medium scalings (R27) are pinned by physics
in ``tests/test_oracle_kop_physics.py``: the field of a uniformly
magnetised sphere and the extinction theorem for plane waves.
"""
