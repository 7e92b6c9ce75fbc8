"""O2: dense complex128 density-matrix simulator (TEST INFRASTRUCTURE ONLY).

Follows §3.3: rho = |Psi><Psi|; a gate acts as rho <- U rho U^dagger
("the gate tensor and its conjugate are applied to the ket (right) and bra
(left) sides"); a channel acts by the Kraus sum Eq.(3)
rho <- sum_k A_k rho A_k^dagger with sum_k A_k^dagger A_k = 1.
Outputs: <b|rho|b>, reduced blocks rho[ket, bra] with other qubits projected,
and Tr(P rho).

rho is stored as a [2]^(2n) tensor: axes 0..n-1 are the ket (row) index, axes
n..2n-1 the bra (column) index, qubit 0 the MSB on both.
"""
from __future__ import annotations

import numpy as np

from .statevector import apply_gate


def _apply_left(rho, M, qubits, n):
    # (M rho)[i, j] = sum_a M[i, a] rho[a, j]  -- ket axes
    return apply_gate(rho, M, qubits)


def _apply_right_dagger(rho, M, qubits, n):
    # (rho M^dagger)[i, j] = sum_b rho[i, b] conj(M[j, b])  -- bra axes with conj(M)
    return apply_gate(rho, np.conj(M), tuple(q + n for q in qubits))


def evolve(oplist) -> np.ndarray:
    n = oplist.nq
    rho = np.zeros((2,) * (2 * n), dtype=np.complex128)
    rho[(0,) * (2 * n)] = 1.0
    for op in oplist.ops:
        if op.kind == "gate":
            U = op.mats[0]
            rho = _apply_right_dagger(_apply_left(rho, U, op.qubits, n), U, op.qubits, n)
        else:
            acc = np.zeros_like(rho)
            for K in op.mats:
                acc += _apply_right_dagger(_apply_left(rho, K, op.qubits, n), K, op.qubits, n)
            rho = acc
    return rho


def as_matrix(rho: np.ndarray) -> np.ndarray:
    n = rho.ndim // 2
    return rho.reshape(2 ** n, 2 ** n)


def probability(rho: np.ndarray, bits) -> complex:
    """<b|rho|b>."""
    n = rho.ndim // 2
    idx = tuple(int(b) for b in bits) * 2
    return complex(rho[idx])


def block(rho: np.ndarray, bits) -> np.ndarray:
    """rho[ket, bra] restricted to the open (-1) qubits, others projected on b;
    row-major ket-major, MSB = lowest open qubit."""
    n = rho.ndim // 2
    sel = tuple(slice(None) if int(b) < 0 else int(b) for b in bits)
    sub = np.array(rho[sel + sel])
    k = sum(1 for b in bits if int(b) < 0)
    return sub.reshape(2 ** k, 2 ** k)


def expectation(rho: np.ndarray, terms):
    """(sum_j c_j Tr(P_j rho), per-term values)."""
    from synth.circuits import PAULI
    n = rho.ndim // 2
    per = []
    for c, term in terms:
        t = rho
        for q, p in term:
            t = _apply_left(t, PAULI[p], (q,), n)
        per.append(complex(np.trace(as_matrix(t))))
    total = sum(c * v for (c, _), v in zip(terms, per))
    return complex(total), np.array(per)
