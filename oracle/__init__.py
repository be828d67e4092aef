"""CPU oracle for the hierarchical block low-rank cavity-radiation hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import anything here.
The product path (`paper_2305_06891_b200`, `include/hm.h`, the CUDA library)
never imports, links or executes this package, and this package never imports
the product path.  The two share only the seeded input generator `synth/`,
which holds none of the method's arithmetic.

Plain, slow, obviously-correct numpy (fp64) written from PAPER.md:
  viewfactor.py  -- eq:Fdef_new_location one-point entry, dense F, row sums and
                    closed-cavity scaling (eq:rowsum, eq:clamped_rowsum, eqn:F_closed),
                    C = I - Lambda F (eq:reflection_matrix), dense solve, flux
                    (eq:qi_new_location), sampled-row (matrix-free) variants.
  tree.py        -- Alg. 1 BuildIndexTree, Alg. 2 BuildBlockTree + admissibility.
  aca.py         -- adaptive cross approximation with partial pivoting (eq:aca, eq:erel)
                    following DESIGN.md reading R10 step by step (probe rows: R30), full
                    pivoting (R31) and QR + SVD recompression (R32).
  cavity.py      -- the cavity operator around the hot path: R, Rbar, S = P^T Rbar P, the flux
                    residual and J^cav (NEXT-1).
  hlu.py         -- the H-LU of C in F's partition: the 4-step recursion on
                    dense blocks with an SVD truncation after every step, its
                    solve and the inverse-factor solve form (reading R27).
  hmatrix.py     -- the oracle's own H-matrix (dense near field + ACA far field) and its
                    block-recursive matrix-vector product.

Parity status per function is listed in DESIGN.md §"Oracle pins".  Unpinned:
none.  The library's H-LU factors are compared with hlu.py block by block at
4 eps (ranks within 2): the two truncate at different points (reading R33).
"""
