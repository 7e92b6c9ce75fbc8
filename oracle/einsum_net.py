"""O3: naive tensor-network contractor (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Builds the circuit's tensor network with its OWN code -- no absorption: every
qubit is a rank-1 tensor, every 1-qubit gate rank-2 and every 2-qubit gate
rank-4, wired in gate order (§3.1; Fig. tensor_notations /
circuit_tensor_network).  Closures:
  * amplitude: open legs closed with <b_q| (Eq.(1));
  * marginal slice: legs with b_q = -1 stay open;
  * expectation by conjugate: U|0>, Pauli tensors, then the conjugate network
    (Table 1, Eq.(2)) -- here as ket copy (U) and bra copy (U*)
    joined through P;
  * noisy: gate tensors on ket (U) and bra (U*) sides, Kraus tensors
    N = sum_k K (x) K* touching both sides (rank 4 / rank 8), closed by
    projection or by joining ket and bra legs through an observable (trace,
    P:L254, Fig. dm_exp_val_trace).

Contraction: one pairwise ``numpy.tensordot`` at a time along its OWN
order -- a min-result-size greedy with a small set of seeded restarts, cheapest
by multiply-add count kept -- and its own memory sub-slicing whose partial
results are summed ("slicing some of the tensor network indices").

Slice-subset mode: reads the GPU plan's sliced wire NAMES (side, qubit,
segment) as data, fixes the matching wires of this network to the slice's
mixed-radix digits (first sliced wire = most significant), and contracts.

Wire naming (shared convention, DESIGN.md §3 R7): wire (side, q, s) is the
state of qubit q on that side right after its s-th two-qubit operation (s = 0:
the initial state), before any later one-qubit operation.  Here such a wire has
label (side, q, s, 0); one-qubit ops append sub-positions 1, 2, ...
"""
from __future__ import annotations

import math
from collections import defaultdict

import numpy as np

E = (np.array([1.0, 0.0], dtype=np.complex128), np.array([0.0, 1.0], dtype=np.complex128))


class Network:
    def __init__(self):
        self.tensors = []      # list of (ndarray, [labels])
        self.open = []         # ordered open labels (output axes)

    def add(self, arr, labels):
        arr = np.asarray(arr, dtype=np.complex128)
        assert arr.ndim == len(labels)
        self.tensors.append((arr, list(labels)))


# ---------------------------------------------------------------------------
# network construction
# ---------------------------------------------------------------------------


class _Wires:
    """Per-qubit wire counters shared by the ket and bra sides."""

    def __init__(self, n, sides):
        self.seg = [0] * n
        self.sub = [0] * n
        self.sides = sides

    def cur(self, side, q):
        return (side, q, self.seg[q], self.sub[q])

    def advance1(self, q):
        self.sub[q] += 1

    def advance2(self, q):
        self.seg[q] += 1
        self.sub[q] = 0


def ket_network(oplist, bits) -> Network:
    """<b|U|0> with -1 entries of ``bits`` left open (Eq.(1); §4.4)."""
    n = oplist.nq
    net = Network()
    w = _Wires(n, ("ket",))
    for q in range(n):
        net.add(E[0], [w.cur("ket", q)])
    for op in oplist.ops:
        if op.kind != "gate":
            raise ValueError("ket network takes unitary gates only")
        _add_gate(net, w, "ket", op.mats[0], op.qubits)
    for q in range(n):
        if int(bits[q]) < 0:
            net.open.append(w.cur("ket", q))
        else:
            net.add(E[int(bits[q])], [w.cur("ket", q)])
    return net


def _add_gate(net, w, side, U, qubits, advance=True):
    k = len(qubits)
    ins = [w.cur(side, q) for q in qubits]
    if advance:
        for q in qubits:
            (w.advance1 if k == 1 else w.advance2)(q)
    outs = [w.cur(side, q) for q in qubits]
    net.add(U.reshape((2,) * (2 * k)), outs + ins)


def doubled_network(oplist, closure, cancel=False) -> Network:
    """Ket copy with U, bra copy with U*, Kraus tensors sum_k K (x) K* on both
    sides.  ``closure``:
       ("project", bits)  -> <b|rho|b>, or rho block over the -1 qubits
                            (open axes: ket opens in qubit order, then bra opens);
       ("pauli", term)    -> Tr(P rho) with term = [(q, 'X'|'Y'|'Z'|'I'), ...].
    ``cancel`` is not used: this oracle never drops gates (the GPU path's light
    cone cancellation is checked against it)."""
    from synth.circuits import PAULI
    n = oplist.nq
    net = Network()
    w = _Wires(n, ("ket", "bra"))
    for q in range(n):
        net.add(E[0], [w.cur("ket", q)])
        net.add(E[0], [w.cur("bra", q)])
    for op in oplist.ops:
        k = len(op.qubits)
        kin = [w.cur("ket", q) for q in op.qubits]
        bin_ = [w.cur("bra", q) for q in op.qubits]
        for q in op.qubits:
            (w.advance1 if k == 1 else w.advance2)(q)
        kout = [w.cur("ket", q) for q in op.qubits]
        bout = [w.cur("bra", q) for q in op.qubits]
        if op.kind == "gate":
            U = op.mats[0]
            net.add(U.reshape((2,) * (2 * k)), kout + kin)
            net.add(np.conj(U).reshape((2,) * (2 * k)), bout + bin_)
        else:
            d = 2 ** k
            N = np.zeros((d, d, d, d), dtype=np.complex128)   # [ko, ki, bo, bi]
            for K in op.mats:
                N += np.einsum("ac,bd->acbd", K, np.conj(K))
            N = N.reshape((2,) * (4 * k))                       # ko.., ki.., bo.., bi..
            ko = list(range(0, k)); ki = list(range(k, 2 * k))
            bo = list(range(2 * k, 3 * k)); bi = list(range(3 * k, 4 * k))
            N = np.transpose(N, ko + bo + ki + bi)
            net.add(N, kout + bout + kin + bin_)
    kind, arg = closure
    if kind == "project":
        bits = arg
        opens_k, opens_b = [], []
        for q in range(n):
            if int(bits[q]) < 0:
                opens_k.append(w.cur("ket", q))
                opens_b.append(w.cur("bra", q))
            else:
                net.add(E[int(bits[q])], [w.cur("ket", q)])
                net.add(E[int(bits[q])], [w.cur("bra", q)])
        net.open = opens_k + opens_b
    elif kind == "pauli":
        P = {q: PAULI[p] for q, p in arg}
        for q in range(n):
            M = P.get(q, PAULI["I"])
            # Tr(P rho) = sum_{i,j} P[j, i] rho[i, j]: tensor T[i_ket, j_bra] = P[j, i]
            net.add(M.T, [w.cur("ket", q), w.cur("bra", q)])
    else:
        raise ValueError(kind)
    return net


# ---------------------------------------------------------------------------
# contraction order: own greedy with seeded restarts
# ---------------------------------------------------------------------------


def greedy_path(label_sets, restarts=16, seed=12345, tau=0.6):
    """Pairwise SSA path [(i, j), ...] over tensors with the given label sets.
    Score of a candidate pair: log2|out| - log2(|A| + |B|) (min-result-size greedy);
    restart 0 is deterministic, restarts r > 0 add Gumbel noise of scale tau.
    The path with the fewest multiply-adds (sum_steps 2^|A u B|) wins."""
    best = None
    for r in range(restarts):
        rng = np.random.default_rng(seed + r) if r > 0 else None
        path, macs, mx = _greedy_once(label_sets, rng, tau)
        key = (macs, mx, r)
        if best is None or key < best[0]:
            best = (key, path)
    return best[1], best[0][0], best[0][1]


def _greedy_once(label_sets, rng, tau):
    active = {i: frozenset(s) for i, s in enumerate(label_sets)}
    where = defaultdict(set)
    for i, s in active.items():
        for l in s:
            where[l].add(i)
    nxt = len(label_sets)
    path, macs, mx = [], 0, 0
    while len(active) > 1:
        cands = set()
        for l, ids in where.items():
            if len(ids) == 2:
                a, b = sorted(ids)
                cands.add((a, b))
        if not cands:  # disconnected: outer product of the two smallest
            ids = sorted(active, key=lambda i: (len(active[i]), i))[:2]
            cands = {tuple(sorted(ids))}
        best = None
        for a, b in sorted(cands):
            A, B = active[a], active[b]
            out = A ^ B
            score = len(out) - math.log2(2.0 ** len(A) + 2.0 ** len(B))
            if rng is not None:
                score -= tau * (-math.log(-math.log(rng.random() + 1e-300) + 1e-300))
            if best is None or score < best[0]:
                best = (score, a, b)
        _, a, b = best
        A, B = active.pop(a), active.pop(b)
        out = A ^ B
        macs += 2 ** len(A | B)
        mx = max(mx, 2 ** len(out))
        for l in A:
            where[l].discard(a)
        for l in B:
            where[l].discard(b)
        for l in out:
            where[l].add(nxt)
        for l in (A & B):
            if not where[l]:
                del where[l]
        active[nxt] = out
        path.append((a, b))
        nxt += 1
    return path, macs, mx


def _intermediates(label_sets, path):
    sets = [frozenset(s) for s in label_sets]
    outs = []
    for a, b in path:
        o = sets[a] ^ sets[b]
        sets.append(o)
        outs.append(o)
    return outs


def choose_subslices(label_sets, path, cap_elems, protected):
    """Own memory slicer: fix the wire shared by most over-cap intermediates until
    every intermediate has <= cap_elems entries."""
    fixed = []
    while True:
        sets = [frozenset(l for l in s if l not in fixed) for s in label_sets]
        outs = _intermediates(sets, path)
        big = [o for o in outs if 2 ** len(o) > cap_elems]
        if not big:
            return fixed
        count = defaultdict(int)
        for o in big:
            for l in o:
                if l not in protected:
                    count[l] += 1
        if not count:
            return fixed
        l = min(count, key=lambda x: (-count[x], str(x)))
        fixed.append(l)


# ---------------------------------------------------------------------------
# evaluation
# ---------------------------------------------------------------------------


def _fix(tensors, assignment):
    out = []
    for arr, labels in tensors:
        for l, v in assignment.items():
            if l in labels:
                ax = labels.index(l)
                arr = np.take(arr, v, axis=ax)
                labels = labels[:ax] + labels[ax + 1:]
        out.append((arr, labels))
    return out


def _run_path(tensors, path):
    pool = list(tensors)
    for a, b in path:
        A, la = pool[a]
        B, lb = pool[b]
        shared = [l for l in la if l in lb]
        C = np.tensordot(A, B, axes=([la.index(l) for l in shared], [lb.index(l) for l in shared]))
        lc = [l for l in la if l not in shared] + [l for l in lb if l not in shared]
        pool.append((C, lc))
        pool[a] = pool[b] = None
    return pool[-1]


def contract(net: Network, fixed=None, restarts=16, seed=12345, cap_elems=2 ** 26, path=None):
    """Value of the network (ndarray over ``net.open``, or a complex scalar)."""
    tensors = _fix(net.tensors, fixed or {})
    if len(tensors) == 1:
        path = []
    elif path is None:
        path, _, _ = greedy_path([t[1] for t in tensors], restarts, seed)
    sub = choose_subslices([t[1] for t in tensors], path, cap_elems, set(net.open))
    total = None
    for x in range(2 ** len(sub)):
        assign = {l: (x >> (len(sub) - 1 - i)) & 1 for i, l in enumerate(sub)}
        arr, labels = _run_path(_fix(tensors, assign), path) if path else _fix(tensors, assign)[0]
        if net.open:
            arr = np.transpose(arr, [labels.index(l) for l in net.open])
        total = arr if total is None else total + arr
    if not net.open:
        return complex(total)
    return np.array(total).reshape(-1)


def label_of(wire) -> tuple:
    """Plan-JSON wire record {side, qubit, segment} -> this network's label."""
    return (wire["side"], int(wire["qubit"]), int(wire["segment"]), 0)


def slice_assignment(sliced_wires, slice_id):
    """Mixed radix (all extents 2) with the first sliced wire the most significant digit."""
    S = len(sliced_wires)
    return {label_of(w): (int(slice_id) >> (S - 1 - i)) & 1 for i, w in enumerate(sliced_wires)}


def slice_values(net: Network, sliced_wires, slice_ids, restarts=16, seed=12345, cap_elems=2 ** 26):
    """Per-slice values for the given slice ids of a plan whose sliced wires are
    ``sliced_wires`` (list of {side, qubit, segment} records, MSB first)."""
    labels_all = {l for _, ls in net.tensors for l in ls}
    for w in sliced_wires:
        if label_of(w) not in labels_all:
            raise KeyError(f"sliced wire {w} not in oracle network")
    first = _fix(net.tensors, slice_assignment(sliced_wires, 0))
    path, _, _ = greedy_path([t[1] for t in first], restarts, seed) if len(first) > 1 else ([], 0, 0)
    return [contract(net, slice_assignment(sliced_wires, s), path=path, cap_elems=cap_elems)
            for s in slice_ids]


def timed_sample(net: Network, fixed, budget_s=20.0, restarts=8, seed=12345, cap_elems=2 ** 26):
    """Bounded CPU-baseline sample (bench.py only): contract the memory sub-slices of the
    network with ``fixed`` wires in order until ``budget_s`` elapses.
    Returns (elapsed seconds, sub-slices done, sub-slices total, path search seconds)."""
    import time
    t0 = time.perf_counter()
    tensors = _fix(net.tensors, fixed or {})
    path, _, _ = greedy_path([t[1] for t in tensors], restarts, seed)
    sub = choose_subslices([t[1] for t in tensors], path, cap_elems, set(net.open))
    t1 = time.perf_counter()
    done = 0
    for x in range(2 ** len(sub)):
        assign = {l: (x >> (len(sub) - 1 - i)) & 1 for i, l in enumerate(sub)}
        _run_path(_fix(tensors, assign), path)
        done += 1
        if time.perf_counter() - t1 > budget_s:
            break
    return time.perf_counter() - t1, done, 2 ** len(sub), t1 - t0


def subslice_plan(net: Network, fixed, restarts=8, seed=12345, cap_elems=2 ** 26):
    """Setup of a timed oracle run (bench.py only): the network with ``fixed`` wires, its
    own greedy path and its own memory sub-slicing.  Returns (tensors, path, sub) for
    contract_subslice; the value of the fixed network is the sum over x in [0, 2^len(sub))."""
    tensors = _fix(net.tensors, fixed or {})
    path, _, _ = greedy_path([t[1] for t in tensors], restarts, seed)
    sub = choose_subslices([t[1] for t in tensors], path, cap_elems, set(net.open))
    return tensors, path, sub


def contract_subslice(tensors, path, sub, x):
    """Value of memory sub-slice x of a subslice_plan (scalar networks: complex)."""
    assign = {l: (x >> (len(sub) - 1 - i)) & 1 for i, l in enumerate(sub)}
    arr, _ = _run_path(_fix(tensors, assign), path)
    return complex(arr) if np.ndim(arr) == 0 else arr


# convenience front-ends ----------------------------------------------------


def amplitude(oplist, bits, **kw) -> complex:
    return contract(ket_network(oplist, bits), **kw)


def amplitudes(oplist, bits, **kw) -> np.ndarray:
    return contract(ket_network(oplist, bits), **kw)


def noisy_block(oplist, bits, **kw):
    """<b|rho|b> (no open qubit) or the rho block over the -1 qubits (ket-major)."""
    v = contract(doubled_network(oplist, ("project", bits)), **kw)
    if isinstance(v, complex):
        return v
    k = int(round(math.log2(v.size) / 2))
    return v.reshape(2 ** k, 2 ** k)


def expectation(oplist, terms, **kw):
    """(sum_j c_j Tr(P_j rho), per-term values) by the bra-ket network (Eq.(2))."""
    per = []
    for c, term in terms:
        per.append(contract(doubled_network(oplist, ("pauli", term)), **kw))
    total = sum(c * v for (c, _), v in zip(terms, per))
    return complex(total), np.array(per)
