"""Pins for the CPU oracle against what the paper and the mathematics fix
(closed forms, invariants, brute force on tiny inputs, the paper's worked
example).  These run on CPU (-m "not gpu")."""
import math
import os

import numpy as np
import pytest

from oracle import densitymatrix as dm
from oracle import einsum_net as tn
from oracle import lightcone as lc
from oracle import statevector as sv
from synth import circuits as C

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------------------
# brute force: full 2^n x 2^n unitary from Kronecker products (independent arithmetic)
# ---------------------------------------------------------------------------


def _full_matrix(U, qubits, n):
    """Embed a k-qubit gate into 2^n x 2^n by explicit basis enumeration."""
    N = 2 ** n
    k = len(qubits)
    M = np.zeros((N, N), dtype=np.complex128)
    for col in range(N):
        bits = [(col >> (n - 1 - q)) & 1 for q in range(n)]
        j = 0
        for q in qubits:
            j = 2 * j + bits[q]
        for i in range(2 ** k):
            nb = list(bits)
            for t, q in enumerate(qubits):
                nb[q] = (i >> (k - 1 - t)) & 1
            row = 0
            for b in nb:
                row = 2 * row + b
            M[row, col] += U[i, j]
    return M


def _brute_state(oplist):
    n = oplist.nq
    psi = np.zeros(2 ** n, dtype=np.complex128)
    psi[0] = 1
    for op in oplist.ops:
        psi = _full_matrix(op.mats[0], op.qubits, n) @ psi
    return psi


def _brute_rho(oplist):
    n = oplist.nq
    rho = np.zeros((2 ** n, 2 ** n), dtype=np.complex128)
    rho[0, 0] = 1
    for op in oplist.ops:
        Ms = [_full_matrix(K, op.qubits, n) for K in op.mats]
        rho = sum(M @ rho @ M.conj().T for M in Ms)
    return rho


@pytest.mark.parametrize("seed", range(4))
def test_statevector_matches_kronecker_bruteforce(seed):
    c = C.random_circuit(5, 6, seed)
    np.testing.assert_allclose(sv.evolve(c), _brute_state(c), atol=1e-13)


def test_bell_golden():
    psi = sv.evolve(C.bell())
    for kind, arg, val in _golden_rows("bell.txt"):
        if kind == "amp":
            assert abs(sv.amplitude(psi, [int(ch) for ch in arg]) - float(val)) < 1e-15
        else:
            term = [(q, p) for q, p in enumerate(arg) if p != "I"]
            tot, _ = sv.expectation(psi, 2, [(1.0, term)])
            assert abs(tot - float(val)) < 1e-15


@pytest.mark.parametrize("n", [2, 3, 5, 8, 12])
def test_ghz_closed_form(n):
    psi = sv.evolve(C.ghz(n))
    ref = np.zeros(2 ** n)
    ref[0] = ref[-1] = 1 / math.sqrt(2)
    np.testing.assert_allclose(psi, ref, atol=1e-15)


def ghz_qft_closed(n):
    N = 2 ** n
    k = np.arange(N)
    return (1 + np.exp(-2j * np.pi * k / N)) / math.sqrt(2 * N)


def test_ghz_qft_closed_form():
    """BASELINE config 1: a_k = (1 + e^{-2 pi i k/256}) / sqrt(512)."""
    psi = sv.evolve(C.ghz_qft(8))
    np.testing.assert_allclose(psi, ghz_qft_closed(8), atol=1e-14)


@pytest.mark.parametrize("x", [0, 1, 37, 200])
def test_qft_basis_closed_form(x):
    n, N = 8, 256
    psi = sv.evolve(C.basis_qft(n, x))
    k = np.arange(N)
    np.testing.assert_allclose(psi, np.exp(2j * np.pi * x * k / N) / 16, atol=1e-14)


def test_unitarity_of_catalogue():
    mats = [C.H, C.X, C.Y, C.Z, C.SQRT_X, C.SQRT_Y, C.SQRT_W, C.CX, C.SWAP,
            C.fsim(math.pi / 2, math.pi / 6), C.cphase(0.3), C.rzz(0.2), C.rx(0.6)]
    for U in mats:
        np.testing.assert_allclose(U.conj().T @ U, np.eye(U.shape[0]), atol=1e-15)


def test_fsim_spec_example():
    """fSim(pi/2, 0)|01> = -i|10>."""
    v = C.fsim(math.pi / 2, 0) @ np.array([0, 1, 0, 0])
    np.testing.assert_allclose(v, [0, 0, -1j, 0], atol=1e-15)


def test_norm_and_porter_thomas():
    """Random grid circuit (4x5, m=10): sum |a|^2 = 1 and Porter-Thomas moment
    E[(N p)^2] = 2 (exponential distribution) within a window."""
    psi = sv.evolve(C.grid_rqc(4, 5, 10, seed=0))
    p = np.abs(psi) ** 2
    assert abs(p.sum() - 1) < 1e-12
    x = p * p.size
    assert 1.9 < np.mean(x ** 2) < 2.1
    assert 0.085 < np.mean(x < 0.1) < 0.105     # 1 - e^{-0.1} = 0.0952


def test_sycamore_generator_counts():
    """E9: 53 qubits, patterns 24/19/23/20, 215 / 301 two-qubit gates at m=10 / 14."""
    sites = C.grid_sites(C.SYCAMORE_ROWS, C.SYCAMORE_DROPPED)
    assert len(sites) == 53
    pats = C.coupler_patterns(sites)
    assert [len(pats[k]) for k in "ABCD"] == [24, 19, 23, 20]
    for v in pats.values():
        qs = [q for e in v for q in e]
        assert len(qs) == len(set(qs))
    assert C.sycamore53(10).n2q() == 215
    assert C.sycamore53(14).n2q() == 301


# ---------------------------------------------------------------------------
# density matrix: Kraus sets and closed forms
# ---------------------------------------------------------------------------

CHANNELS = {
    "dep1": C.depolarizing1(0.07),
    "dep2": C.depolarizing2(0.05),
    "ad": C.amplitude_damping(0.13),
    "deph": C.dephasing(0.2),
}


@pytest.mark.parametrize("name", sorted(CHANNELS))
def test_kraus_completeness(name):
    Ks = CHANNELS[name]
    S = sum(K.conj().T @ K for K in Ks)
    np.testing.assert_allclose(S, np.eye(S.shape[0]), atol=1e-15)


@pytest.mark.parametrize("k", [1, 3, 7])
def test_depolarizing_closed_form(k):
    p = 0.05
    c = C.OpList(1)
    for _ in range(k):
        c.kraus(C.depolarizing1(p), 0)
    rho = dm.evolve(c)
    z, _ = dm.expectation(rho, [(1.0, [(0, "Z")])])
    assert abs(z - (1 - p) ** k) < 1e-14


@pytest.mark.parametrize("k", [1, 4, 25])
def test_hh_depolarizing_sequence(k):
    """H-H cycles with depolarizing after each H: <Z> = (1-p)^{2k}."""
    p = 0.01
    c = C.OpList(1)
    for _ in range(k):
        for _ in range(2):
            c.gate(C.H, 0).kraus(C.depolarizing1(p), 0)
    z, _ = dm.expectation(dm.evolve(c), [(1.0, [(0, "Z")])])
    assert abs(z - (1 - p) ** (2 * k)) < 1e-13


@pytest.mark.parametrize("k", [1, 5])
def test_amplitude_damping_closed_form(k):
    g = 0.1
    c = C.OpList(1).gate(C.X, 0)
    for _ in range(k):
        c.kraus(C.amplitude_damping(g), 0)
    rho = dm.evolve(c)
    assert abs(dm.probability(rho, [1]) - (1 - g) ** k) < 1e-15
    z, _ = dm.expectation(rho, [(1.0, [(0, "Z")])])
    assert abs(z - (1 - 2 * (1 - g) ** k)) < 1e-14


def test_dephasing_closed_form():
    p, k = 0.1, 4
    c = C.OpList(1).gate(C.H, 0)
    for _ in range(k):
        c.kraus(C.dephasing(p), 0)
    x, _ = dm.expectation(dm.evolve(c), [(1.0, [(0, "X")])])
    assert abs(x - (1 - 2 * p) ** k) < 1e-14


def test_dep2_is_depolarizing_to_identity():
    """2q depolarizing: rho -> (1-p) rho + p I/4 (reading R5)."""
    rng = np.random.default_rng(3)
    A = rng.normal(size=(4, 4)) + 1j * rng.normal(size=(4, 4))
    rho = A @ A.conj().T
    rho /= np.trace(rho)
    p = 0.3
    out = sum(K @ rho @ K.conj().T for K in C.depolarizing2(p))
    np.testing.assert_allclose(out, (1 - p) * rho + p * np.eye(4) / 4, atol=1e-15)


@pytest.mark.parametrize("seed", range(3))
def test_density_matrix_bruteforce_and_invariants(seed):
    rng = np.random.default_rng(seed)
    c = C.random_circuit(4, 4, seed)
    noisy = C.OpList(4)
    for op in c.ops:
        noisy.ops.append(op)
        noisy.kraus(C.depolarizing1(0.05), op.qubits[0])
        noisy.kraus(C.amplitude_damping(0.07), op.qubits[-1])
        if len(op.qubits) == 2 and rng.random() < 0.5:
            noisy.kraus(C.depolarizing2(0.04), *op.qubits)
    rho = dm.as_matrix(dm.evolve(noisy))
    np.testing.assert_allclose(rho, _brute_rho(noisy), atol=1e-14)
    assert abs(np.trace(rho) - 1) < 1e-13
    np.testing.assert_allclose(rho, rho.conj().T, atol=1e-15)
    assert np.linalg.eigvalsh(rho).min() > -1e-13


def test_density_matrix_reduces_to_pure():
    c = C.random_circuit(5, 5, 9)
    psi = sv.evolve(c)
    rho = dm.as_matrix(dm.evolve(c))
    np.testing.assert_allclose(rho, np.outer(psi, psi.conj()), atol=1e-14)


# ---------------------------------------------------------------------------
# O3 naive contractor
# ---------------------------------------------------------------------------


def test_cat_state_paper_example():
    """The paper's §4.4 worked example on 60 qubits (golden fixture)."""
    c = C.cat_state(60)
    for row in _golden_rows("cat60_marginal.txt"):
        other = int(row[0])
        ref = np.array([float(v) for v in row[1:]])
        bits = [other] * 60
        bits[2] = bits[47] = -1
        v = tn.amplitudes(c, bits, restarts=2)
        assert abs(np.linalg.norm(v) - 1 / math.sqrt(2)) < 1e-14   # |Psi> = (|0..0> + |1..1>)/sqrt2
        np.testing.assert_allclose(v / np.linalg.norm(v), ref, atol=1e-14)
    bits = [0] * 60
    bits[5] = 1
    bits[2] = bits[47] = -1
    assert np.abs(tn.amplitudes(c, bits, restarts=2)).max() < 1e-15


@pytest.mark.parametrize("seed", range(3))
def test_einsum_matches_bruteforce(seed):
    c = C.random_circuit(7, 8, seed)
    psi = _brute_state(c)
    rng = np.random.default_rng(seed)
    for _ in range(3):
        bits = rng.integers(0, 2, size=7)
        assert abs(tn.amplitude(c, bits, restarts=3) - psi[sv.index_of(bits)]) < 1e-13
    bits = [-1] * 7
    np.testing.assert_allclose(tn.amplitudes(c, bits, restarts=3), psi, atol=1e-13)
    bits = list(rng.integers(0, 2, size=7))
    bits[1] = bits[4] = -1
    np.testing.assert_allclose(tn.amplitudes(c, bits, restarts=3), sv.amplitudes(psi, bits), atol=1e-13)


def test_einsum_ghz_qft_closed_form():
    v = tn.amplitudes(C.ghz_qft(8), [-1] * 8, restarts=3)
    np.testing.assert_allclose(v, ghz_qft_closed(8), atol=1e-14)


def test_einsum_slice_sum_identity():
    """Sum over every assignment of fixed wires equals the unsliced value."""
    c = C.grid_rqc(3, 3, 6, seed=1)
    bits = [0, 1, 1, 0, 1, 0, 0, 1, 1]
    net = tn.ket_network(c, bits)
    full = tn.contract(net, restarts=2)
    wires = [{"side": "ket", "qubit": 4, "segment": 1}, {"side": "ket", "qubit": 1, "segment": 2},
             {"side": "ket", "qubit": 7, "segment": 1}]
    vals = tn.slice_values(net, wires, range(8), restarts=2)
    assert abs(sum(vals) - full) < 1e-14
    assert abs(full - sv.amplitude(sv.evolve(c), bits)) < 1e-14
    # forced memory sub-slicing gives the same value
    assert abs(tn.contract(net, restarts=2, cap_elems=64) - full) < 1e-14


@pytest.mark.parametrize("seed", range(2))
def test_einsum_doubled_network_matches_density_matrix(seed):
    rng = np.random.default_rng(100 + seed)
    c = C.random_circuit(4, 5, seed)
    noisy = C.OpList(4)
    for op in c.ops:
        noisy.ops.append(op)
        if len(op.qubits) == 2:
            noisy.kraus(C.depolarizing2(0.05), *op.qubits)
        for q in op.qubits:
            noisy.kraus(C.depolarizing1(0.02), q).kraus(C.amplitude_damping(0.07), q)
    rho = dm.evolve(noisy)
    bits = rng.integers(0, 2, size=4)
    assert abs(tn.noisy_block(noisy, bits, restarts=2) - dm.probability(rho, bits)) < 1e-14
    bits = list(bits)
    bits[0] = bits[2] = -1
    np.testing.assert_allclose(tn.noisy_block(noisy, bits, restarts=2), dm.block(rho, bits), atol=1e-14)
    terms = [(0.5, [(0, "Z")]), (1.5, [(1, "X"), (3, "Y")]), (-0.25, [(2, "Z"), (3, "Z")])]
    tot, per = tn.expectation(noisy, terms, restarts=2)
    tot_ref, per_ref = dm.expectation(rho, terms)
    np.testing.assert_allclose(per, per_ref, atol=1e-14)
    # trace preservation of the full doubled network: Tr rho = 1
    one, _ = tn.expectation(noisy, [(1.0, [])], restarts=2)
    assert abs(one - 1) < 1e-13


def test_einsum_pure_expectation_matches_statevector():
    c = C.random_circuit(6, 6, 4)
    psi = sv.evolve(c)
    terms = [(1.0, [(0, "Z"), (1, "Z")]), (0.3, [(2, "X")]), (0.7, [(3, "Y"), (5, "X")])]
    tot, per = tn.expectation(c, terms, restarts=2)
    tot_ref, per_ref = sv.expectation(psi, 6, terms)
    np.testing.assert_allclose(per, per_ref, atol=1e-14)
    assert abs(tot - tot_ref) < 1e-14


def test_bell_expectations_spec():
    """Bell Z(x)Z = 1 and H then Z = 0."""
    tot, _ = tn.expectation(C.bell(), [(1.0, [(0, "Z"), (1, "Z")])], restarts=1)
    assert abs(tot - 1) < 1e-15
    tot, _ = tn.expectation(C.OpList(1).gate(C.H, 0), [(1.0, [(0, "Z")])], restarts=1)
    assert abs(tot) < 1e-15


# ---------------------------------------------------------------------------
# QAOA: closed form (p=1) and light cone (O4)
# ---------------------------------------------------------------------------


def _cube_graph_edges():
    """Q3 cube graph: 3-regular, triangle-free, 8 nodes."""
    return sorted((a, b) for a in range(8) for b in range(a + 1, 8) if bin(a ^ b).count("1") == 1)


def test_qaoa_p1_closed_form():
    """<Z_u Z_v> = sin(4b) sin(2g) cos^{D-1}(2g) for D-regular triangle-free graphs
    (Wang, Hadfield, Jiang, Rieffel, PRA 97 022304 (2018)) with our
    U_C = prod exp(-i g ZZ), U_B = prod exp(-i b X)."""
    edges = _cube_graph_edges()
    g, b = 0.37, 0.81
    c = C.qaoa_circuit(8, edges, [g], [b])
    psi = sv.evolve(c)
    ref = math.sin(4 * b) * math.sin(2 * g) * math.cos(2 * g) ** 2
    _, per = sv.expectation(psi, 8, C.maxcut_terms(edges))
    np.testing.assert_allclose(per.real, ref, atol=1e-14)
    _, per_lc = lc.expectation(c, C.maxcut_terms(edges))
    np.testing.assert_allclose(np.real(per_lc), ref, atol=1e-14)
    _, per_tn = tn.expectation(c, C.maxcut_terms(edges)[:3], restarts=2)
    np.testing.assert_allclose(per_tn.real, ref, atol=1e-14)


def test_lightcone_matches_full_statevector():
    edges = C.regular_graph(3, 14, seed=1)
    c = C.qaoa_circuit(14, edges, C.QAOA_GAMMAS, C.QAOA_BETAS)
    terms = C.maxcut_terms(edges)
    _, per_ref = sv.expectation(sv.evolve(c), 14, terms)
    _, per = lc.expectation(c, terms)
    np.testing.assert_allclose(per, per_ref, atol=1e-13)


def test_qaoa40_light_cones_small():
    """E6: p=2 light cones on the 40-qubit 3-regular graph have <= 14 qubits."""
    c, terms = C.qaoa40(0)
    sizes = lc.cone_sizes(c, terms)
    assert max(sizes) <= 14 and len(terms) == 60


# ---------------------------------------------------------------------------
# O6 sampling / O7 wave-function slicing (oracle/sampling.py)
# ---------------------------------------------------------------------------
from oracle import sampling as smp  # noqa: E402


@pytest.mark.parametrize("block", [1, 2, 3])
def test_sampling_is_global_inverse_cdf(block):
    """Sequential block sampling with the lexicographic mass rule equals the inverse CDF of
    |psi|^2 over the state index (qubit 0 = MSB), computed independently with a cumulative
    sum and a binary search."""
    ops = C.random_circuit(8, 10, 11)
    probs = smp.probabilities(sv.evolve(ops))
    cum = np.cumsum(probs)
    rng = np.random.default_rng(5)
    us = [u for u in rng.random(200) if np.min(np.abs(cum - u)) > 1e-9][:100]
    got = smp.sample(probs, 8, us, block)
    for u, row in zip(us, got):
        x = int(np.searchsorted(cum, u, side="right"))
        assert sv.index_of(row) == x


def test_sampling_ghz_and_uniform_closed_forms():
    """GHZ_n: u < 1/2 gives 0^n, else 1^n.  H^n|0>: uniform, so the sample is the binary
    expansion of floor(u 2^n)."""
    n = 6
    probs = smp.probabilities(sv.evolve(C.ghz(n)))
    rows = smp.sample(probs, n, [0.1, 0.49, 0.51, 0.99], block=2)
    assert [list(r) for r in rows] == [[0] * n] * 2 + [[1] * n] * 2
    ops = C.OpList(n)
    for q in range(n):
        ops.gate(C.H, q)
    probs = smp.probabilities(sv.evolve(ops))
    for u in (0.0, 0.3, 0.77, 0.999):
        row = smp.sample(probs, n, [u + 1e-9], block=1)[0]
        assert sv.index_of(row) == int(math.floor((u + 1e-9) * 2 ** n))


def test_marginals_sum_and_prefix_consistency():
    ops = C.random_circuit(7, 8, 3)
    probs = smp.probabilities(sv.evolve(ops))
    assert abs(smp.marginal(probs, 7, []) - 1.0) < 1e-12
    for pre in ([0], [1, 0], [0, 1, 1]):
        tot = sum(smp.marginal(probs, 7, pre + [a]) for a in (0, 1))
        assert abs(tot - smp.marginal(probs, 7, pre)) < 1e-13


@pytest.mark.parametrize("open_q", [[0, 1, 2, 3], [2, 3, 5, 7], list(range(8))])
def test_wf_slicing_expectation_identity(open_q):
    """O7: the sum over all projected bitstrings of the partial expectations equals the
    full <psi|P|psi> (O1) whenever the X / Y support lies in the open set (Z factors on
    projected qubits enter as signs)."""
    ops = C.random_circuit(8, 10, 7)
    psi = sv.evolve(ops)
    terms = [(1.0, [(0, "Z"), (1, "Z")]), (0.5, [(2, "X"), (3, "Y")]), (-0.7, [(3, "Z"), (6, "Z")]), (2.0, [])]
    terms = [t for t in terms if all(q in open_q or ch in "IZ" for q, ch in t[1])]
    tot, per = smp.wf_slice_expectation(psi, 8, terms, open_q)
    tot_ref, per_ref = sv.expectation(psi, 8, terms)
    assert np.max(np.abs(per - per_ref)) < 1e-13 and abs(tot - tot_ref) < 1e-13


def test_wf_slicing_qaoa_p1_closed_form():
    """O7 on QAOA p=1 over the cube graph (3-regular, triangle free):
    <Z_u Z_v> = sin 4b sin 2g cos^2 2g (closed form)."""
    edges = sorted((a, b) for a in range(8) for b in range(a + 1, 8) if bin(a ^ b).count("1") == 1)
    g, b = 0.37, 0.81
    psi = sv.evolve(C.qaoa_circuit(8, edges, [g], [b]))
    terms = C.maxcut_terms(edges)
    _, per = smp.wf_slice_expectation(psi, 8, terms, [0, 1, 2, 3])
    ref = math.sin(4 * b) * math.sin(2 * g) * math.cos(2 * g) ** 2
    assert np.max(np.abs(per - ref)) < 1e-12
