"""O4: per-term backward light cone + O1 (TEST INFRASTRUCTURE ONLY).

<psi|P|psi> with psi = U_G...U_1|0>: a gate whose qubits do not meet the set of
qubits reached so far by the backward sweep commutes past every later kept
gate and past P, and cancels against its conjugate ("ExaTN can intelligently
collapse a tensor and its conjugate"; Eq.(2)).  The kept
gates act on at most |L| qubits; O1 evaluates them exactly on those qubits.
"""
from __future__ import annotations

import numpy as np

from synth.circuits import OpList

from . import statevector as sv


def _is_diagonal(op) -> bool:
    U = op.mats[0]
    return op.kind == "gate" and bool(np.all(np.abs(U - np.diag(np.diag(U))) == 0.0))


def light_cone(oplist, support):
    """Kept op indices (in circuit order) and the final qubit set L.

    Backward sweep.  A maximal run of consecutive diagonal gates is treated as
    one layer of mutually commuting gates: a gate of the run is kept iff it
    meets the set L as it stood *after* the run (closer to P).  A dropped gate
    commutes with the kept gates of its run (all diagonal) and with every later
    kept gate and P (disjoint support), so it cancels against its conjugate.
    (Reading R9 in DESIGN.md.)"""
    L = set(support)
    keep = []
    ops = oplist.ops
    i = len(ops) - 1
    while i >= 0:
        if _is_diagonal(ops[i]):
            j = i
            while j - 1 >= 0 and _is_diagonal(ops[j - 1]):
                j -= 1
            L0 = set(L)
            for t in range(i, j - 1, -1):
                if L0.intersection(ops[t].qubits):
                    keep.append(t)
                    L.update(ops[t].qubits)
            i = j - 1
            continue
        op = ops[i]
        if L.intersection(op.qubits):
            if op.kind != "gate":
                raise ValueError("light-cone oracle handles unitary gates only")
            keep.append(i)
            L.update(op.qubits)
        i -= 1
    return keep[::-1], sorted(L)


def term_value(oplist, term) -> complex:
    support = [q for q, p in term if p != "I"]
    if not support:
        return 1.0 + 0.0j
    keep, L = light_cone(oplist, support)
    relabel = {q: i for i, q in enumerate(L)}
    sub = OpList(len(L))
    for i in keep:
        op = oplist.ops[i]
        sub.gate(op.mats[0], *[relabel[q] for q in op.qubits])
    psi = sv.evolve(sub)
    local = [(relabel[q], p) for q, p in term if p != "I"]
    return complex(sv.expectation(psi, len(L), [(1.0, local)])[0])


def expectation(oplist, terms):
    per = [term_value(oplist, t) for _, t in terms]
    total = sum(c * v for (c, _), v in zip(terms, per))
    return complex(total), per


def cone_sizes(oplist, terms):
    return [len(light_cone(oplist, [q for q, p in t if p != "I"])[1]) for _, t in terms]
