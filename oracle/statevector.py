"""O1: complex128 state-vector simulator (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Computes the exact definitions the method evaluates by contraction:
  * amplitude  a(b) = <b| U_G ... U_1 |0^n>                (Eq.(1))
  * batch      a(b) over the open bits (-1 entries)          (§4.4)
  * expectation sum_j c_j <psi| P_j |psi>, psi = U|0^n>      (Eq.(2))

Algorithm: psi <- e_0; for each gate reshape psi to [2]^n,
contract the gate's input axes with the gate's qubit axes, move the output
axes back.  Qubit 0 is the most significant bit of the state index
(DESIGN.md §3 reading R1).
"""
from __future__ import annotations

import numpy as np


def evolve(oplist) -> np.ndarray:
    """Return psi = U_G ... U_1 |0...0> as a flat complex128 vector of length 2^n."""
    n = oplist.nq
    psi = np.zeros((2,) * n, dtype=np.complex128)
    psi[(0,) * n] = 1.0
    for op in oplist.ops:
        if op.kind != "gate":
            raise ValueError("statevector oracle handles unitary gates only")
        psi = apply_gate(psi, op.mats[0], op.qubits)
    return psi.reshape(-1)


def apply_gate(psi: np.ndarray, U: np.ndarray, qubits) -> np.ndarray:
    """psi[..., i_q, ...] <- sum_j U[i, j] psi[..., j_q, ...] on the gate's qubits."""
    k = len(qubits)
    Ut = U.reshape((2,) * (2 * k))                 # (out_0..out_{k-1}, in_0..in_{k-1})
    out = np.tensordot(Ut, psi, axes=(list(range(k, 2 * k)), list(qubits)))
    return np.moveaxis(out, list(range(k)), list(qubits))


def index_of(bits) -> int:
    """x = sum_q b_q 2^{n-1-q} (qubit 0 = MSB)."""
    x = 0
    for b in bits:
        x = 2 * x + int(b)
    return x


def amplitude(psi: np.ndarray, bits) -> complex:
    return complex(psi[index_of(bits)])


def amplitudes(psi: np.ndarray, bits) -> np.ndarray:
    """Entries of psi with the -1 qubits free; output index MSB = lowest open qubit."""
    n = len(bits)
    t = psi.reshape((2,) * n)
    idx = tuple(slice(None) if int(b) < 0 else int(b) for b in bits)
    return np.array(t[idx]).reshape(-1)


def pauli_apply(psi_flat: np.ndarray, n: int, term) -> np.ndarray:
    """P psi for a Pauli string term = [(q, 'X'|'Y'|'Z'|'I'), ...]."""
    from synth.circuits import PAULI  # Pauli matrices are inputs (synth catalogue)
    t = psi_flat.reshape((2,) * n)
    for q, p in term:
        t = apply_gate(t, PAULI[p], (q,))
    return t.reshape(-1)


def expectation(psi: np.ndarray, n: int, terms):
    """(sum_j c_j <psi|P_j|psi>, per-term values).  terms = [(c_j, [(q, P), ...]), ...]."""
    per = []
    for c, term in terms:
        per.append(complex(np.vdot(psi, pauli_apply(psi, n, term))))
    total = sum(c * v for (c, _), v in zip(terms, per))
    return complex(total), np.array(per)
