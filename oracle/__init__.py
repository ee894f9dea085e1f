"""CPU oracle for the nodal-DG Euler RHS + explicit RK stage (arXiv:1710.03887).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1710_03887_b200``) never imports, links or
executes anything here, and this package never imports the product.  The two
share no code: the oracle builds its own reference element (in mpmath, from a
monomial basis and exact simplex integrals), its own geometry, connectivity,
fluxes and time stepper, all in plain numpy fp64.

Citation key: ``P:n`` = PAPER.md line n, ``S:n`` = SPEC.md line n,
``SURVEY §8(c)`` = the readings of the paper this build fixes (also listed in
DESIGN.md).

Modules
-------
refelem  reference tetrahedron, warp&blend nodes, Dr/Ds/Dt, LIFT
geom     affine geometric factors, normals, Fscale, h
conn     EToE/EToF by face hashing, vmapM/vmapP by coordinates
euler    pressure, Euler fluxes (Eq. 1-2), ghosts (Eq. 3-4, 5-7), LLF flux
rhs      strong-form nodal DG right-hand side f(Q, t)
timestep LSERK4 (Carpenter-Kennedy) and Heun RK2 in 2N-storage form
sensors  point location and nodal evaluation at sensor points       (Table 2)
modal    the paper's modal scheme: orthonormal basis, Gauss rules, weak-form RHS (N3)
analysis DFT amplitude spectra, decay exponent, percent of atmosphere

Parity status: every function is pinned by ``tests/test_oracle_*.py`` except
the items listed as "parity unpinned" in DESIGN.md (absolute accuracy of the
nonlinear 10 % pulses; the per-face vs per-node lambda choice).
"""
