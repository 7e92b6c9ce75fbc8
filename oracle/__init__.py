"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct complex128 reference implementations of what
the hot path computes.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here.  The product path
(``paper_2104_10523_b200``) never imports it, and this package never imports
the product path: the two share no code.  The only shared module is the seeded
input generator ``synth/`` (op lists; none of the method's arithmetic).

Parts (each function cites the passage it follows):
  O1 ``statevector``     -- psi <- U psi, amplitudes <b|U|0> (Eq.(1)),
                            expectation <psi|P|psi> (Eq.(2)).
  O2 ``densitymatrix``   -- rho <- sum_k K rho K^dagger (Eq.(3)).
  O3 ``einsum_net``      -- naive tensor-network contractor on its OWN network
                            and its OWN greedy order, with a
                            slice-subset mode that reads the plan JSON's sliced
                            wire names as data.
  O4 ``lightcone``       -- per-term backward light cone + O1.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``): Bell / GHZ / GHZ->QFT / QFT
closed forms, brute-force Kronecker-matrix evolution on <= 6 qubits, the
paper's cat-state marginal, Kraus completeness, depolarizing /
damping / dephasing closed forms, QAOA p=1 closed form, Porter-Thomas moments,
slice-sum identity.  No function here is "parity unpinned".
"""
