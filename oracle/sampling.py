"""O6 / O7: bit-string sampling and wave-function-slicing expectation on the state vector
(TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

O6 -- direct unbiased bit-string sampling (Table 1 "direct unbiased bit-string sampling",
P:L150: "connecting the quantum circuit tensor network with its conjugate while leaving a
subset of qubit legs open to compute the reduced density matrices for bit-string sampling
and measurement projection").  The qubits are sampled in the order 0, 1, ..., n-1, `block`
at a time.  The probability of a prefix (the sampled qubits set to b, the others traced
out) is the marginal

    P(b_0 .. b_{k-1}) = sum over the unsampled bits of |psi_x|^2      (pure)
                      = sum over the unsampled bits of rho_xx           (noisy)

Decision rule (reading R21), one uniform u in [0, 1) per shot: keep the total
mass m of every prefix that precedes the current one in lexicographic order (qubit 0 the
most significant); for the 2^block extensions a of the current prefix in increasing order,
take the first with m + P(prefix a) > u, else add P(prefix a) to m.  This is the inverse
CDF of |psi|^2 over the state index (DESIGN R1 bit order), computed one block of qubits at
a time -- the probabilities the GPU path returns are exactly these marginals.

O7 -- expectation value by wave-function slicing (Table 1 "expectation value by state
vector slicing"; the five-step workflow): project the N_projected =
n - rank_max qubits outside the open set O to every bitstring p, take the partial state
vector psi_p over O, compute the partial expectation <psi_p| P |psi_p> for each p and sum.
A Pauli string whose X / Y support lies inside O maps each slice to itself; its Z factors
on projected qubits contribute (-1)^{p_q} (reading R22).
"""
from __future__ import annotations

import itertools

import numpy as np

from oracle import statevector as sv


def marginal(probs: np.ndarray, n: int, prefix) -> float:
    """P(qubits 0..len(prefix)-1 = prefix): sum of probs over the unsampled bits."""
    k = len(prefix)
    t = probs.reshape((2,) * n)
    return float(np.sum(t[tuple(int(b) for b in prefix)])) if k else float(np.sum(probs))


def sample(probs: np.ndarray, n: int, uniforms, block: int = 1) -> np.ndarray:
    """O6 on a probability vector over the 2^n state indices (|psi|^2, or diag(rho)).
    Returns one row of n bits per uniform."""
    out = []
    for u in uniforms:
        prefix, m = [], 0.0
        while len(prefix) < n:
            k = min(block, n - len(prefix))
            choice = None
            for a in range(2 ** k):
                ext = prefix + [(a >> (k - 1 - i)) & 1 for i in range(k)]
                p = marginal(probs, n, ext)
                if m + p > u:
                    choice = ext
                    break
                m += p
            if choice is None:  # u beyond the total mass by rounding: the last extension with mass
                for a in reversed(range(2 ** k)):
                    ext = prefix + [(a >> (k - 1 - i)) & 1 for i in range(k)]
                    if marginal(probs, n, ext) > 0:
                        choice = ext
                        break
            prefix = choice
        out.append(prefix)
    return np.array(out, dtype=np.int8)


def probabilities(psi: np.ndarray) -> np.ndarray:
    return np.abs(psi) ** 2


def wf_slice_expectation(psi: np.ndarray, n: int, terms, open_qubits):
    """O7: (sum_j c_j <P_j>, per-term values) accumulated over the wave-function slices.
    terms = [(c, [(q, 'X'|'Y'|'Z'|'I'), ...]), ...]; every X / Y factor must act on an open qubit."""
    open_qubits = sorted(open_qubits)
    proj = [q for q in range(n) if q not in open_qubits]
    per = np.zeros(len(terms), dtype=np.complex128)
    for p in itertools.product((0, 1), repeat=len(proj)):
        bits = [-1] * n
        for q, b in zip(proj, p):
            bits[q] = b
        psi_p = sv.amplitudes(psi, bits)  # partial state vector over the open qubits
        no = len(open_qubits)
        for j, (_, term) in enumerate(terms):
            sign = 1.0
            local = []
            for q, ch in term:
                if q in open_qubits:
                    local.append((open_qubits.index(q), ch))
                elif ch == "Z":
                    sign *= -1.0 if p[proj.index(q)] else 1.0
                elif ch != "I":
                    raise ValueError("X / Y factor on a projected qubit")
            per[j] += sign * np.vdot(psi_p, sv.pauli_apply(psi_p, no, local))
    total = sum(c * v for (c, _), v in zip(terms, per))
    return complex(total), per
