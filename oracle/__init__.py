"""CPU fp64 oracle for the fine-grid solve path of Ferrari & Sigmund (arXiv 1909.13585).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import this package.
The product path (`paper_1909_13585_b200`) never imports it, and this package
never imports the product path; the two share only the seeded input
generators in `workloads/` (which hold none of the method's arithmetic).

What it computes (SURVEY.md 8(c) "Definition"), each function citing its passage:

* `fem`      element matrices K_e0 (standard bilinear Q4 / trilinear H8, exact
             2x2(x2) Gauss of B^T D B; incompatible-mode "Wilson" elements with
             statically condensed bubble modes, NEXT-4) and the centroid-stress geometric
             matrices H_ij used by G_e0[u_e]  (Eq. 2);
* `assemble` sparse K = sum_e E_e A_e^T K0 A_e and G(u) = sum_e Es_e A_e^T G_e0[u_e] A_e
             with Dirichlet rows/cols replaced by identity (K) or zero (G);
* `ebe`      element-by-element products y = K x / G(u) phi on the grid (used
             at sizes where assembly is too large, and in extended precision
             for the refinement residual);
* `solve`    u = K_ff^-1 f_f by sparse direct LU + one refinement step
             (Alg. 1 l.2; Eq. 5 :133-136; Eq. 6 :161-165), and an
             independent multigrid-preconditioned CG for the 3D
             sizes where direct factorisation is infeasible;
* `sens`     adjoint right-hand sides (Eq. 5) and Eq. 4 sensitivities (NEXT-1);
* `mg`       nested hierarchy, bilinear/trilinear prolongation P = I^j_{j+1}
             and the Galerkin product P^T K P (Alg. 2 l.5).

Parity status: every function above is pinned in tests/test_oracle_pins.py
(closed forms, exact patch solutions, beam theory, Euler buckling, brute
force, paper-printed DOF counts).  Parity unpinned: MG iteration counts
(PAPER.md:758 gives ranges for other designs and another stopping rule).
"""
