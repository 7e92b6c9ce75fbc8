"""Seeded synthetic workload generators (shared INPUT module).

This module is the only code shared by the CUDA path (through the C-ABI) and
the CPU oracle (``oracle/``).  It holds NO arithmetic of the method: it only
produces *op lists* -- ordered gates ``U`` (2^k x 2^k, k in {1,2}) and Kraus
sets ``{K_j}`` with the qubits they act on -- which both sides consume and turn
into tensor networks independently (SURVEY.md §8(c) "Shared test input").

Gate matrices follow SURVEY.md §8(d) "Gate matrices for the synthetic
generators"; channels follow the readings listed in DESIGN.md §3
(depolarizing, amplitude damping, dephasing).

Conventions:
  * a gate matrix is row-major in the basis |q_{qubits[0]} q_{qubits[1]}>,
    qubits[0] is the most significant bit;
  * qubit 0 is the MSB of a state index.

Workload shapes (paper: Sycamore random circuits P:L443-467, cat state
P:L512-548, noisy circuits §3.3; configs from BASELINE.json).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# op list
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class Op:
    kind: str                 # "gate" or "kraus"
    qubits: tuple             # 1 or 2 distinct qubit indices
    mats: tuple               # gate: (U,), kraus: (K_0, ..., K_{m-1}); complex128 2^k x 2^k
    name: str = ""


@dataclass
class OpList:
    nq: int
    ops: list = field(default_factory=list)

    def gate(self, U, *qubits, name=""):
        U = np.asarray(U, dtype=np.complex128)
        self.ops.append(Op("gate", tuple(int(q) for q in qubits), (U,), name))
        return self

    def kraus(self, Ks, *qubits, name=""):
        Ks = tuple(np.asarray(K, dtype=np.complex128) for K in Ks)
        self.ops.append(Op("kraus", tuple(int(q) for q in qubits), Ks, name))
        return self

    @property
    def noisy(self) -> bool:
        return any(op.kind == "kraus" for op in self.ops)

    def n2q(self) -> int:
        return sum(1 for op in self.ops if len(op.qubits) == 2)

    def to_text(self) -> str:
        """Plain text form (one op per line) for fixtures."""
        lines = [f"nq {self.nq}"]
        for op in self.ops:
            vals = " ".join(f"{z.real:.17g},{z.imag:.17g}" for M in op.mats for z in M.ravel())
            lines.append(f"{op.kind} {op.name or '-'} {len(op.mats)} {' '.join(map(str, op.qubits))} : {vals}")
        return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# gate and channel catalogue (inputs)
# ---------------------------------------------------------------------------

S2 = 1.0 / math.sqrt(2.0)

I2 = np.eye(2, dtype=np.complex128)
X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
Y = np.array([[0, -1j], [1j, 0]], dtype=np.complex128)
Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
H = S2 * np.array([[1, 1], [1, -1]], dtype=np.complex128)
PAULI = {"I": I2, "X": X, "Y": Y, "Z": Z}

SQRT_X = S2 * np.array([[1, -1j], [-1j, 1]], dtype=np.complex128)
SQRT_Y = S2 * np.array([[1, -1], [1, 1]], dtype=np.complex128)
_SQI = np.exp(1j * math.pi / 4)          # sqrt(i)
_SQMI = np.exp(-1j * math.pi / 4)        # sqrt(-i)
SQRT_W = S2 * np.array([[1, -_SQI], [_SQMI, 1]], dtype=np.complex128)
SYC_1Q = (SQRT_X, SQRT_Y, SQRT_W)
SYC_1Q_NAMES = ("sqrtX", "sqrtY", "sqrtW")

CX = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]], dtype=np.complex128)
SWAP = np.array([[1, 0, 0, 0], [0, 0, 1, 0], [0, 1, 0, 0], [0, 0, 0, 1]], dtype=np.complex128)


def fsim(theta: float, phi: float) -> np.ndarray:
    c, s = math.cos(theta), math.sin(theta)
    return np.array([[1, 0, 0, 0],
                     [0, c, -1j * s, 0],
                     [0, -1j * s, c, 0],
                     [0, 0, 0, np.exp(-1j * phi)]], dtype=np.complex128)


def cphase(t: float) -> np.ndarray:
    return np.diag([1, 1, 1, np.exp(1j * t)]).astype(np.complex128)


def rzz(g: float) -> np.ndarray:
    """exp(-i g Z(x)Z)."""
    return np.diag([np.exp(-1j * g), np.exp(1j * g), np.exp(1j * g), np.exp(-1j * g)]).astype(np.complex128)


def rx(b: float) -> np.ndarray:
    """exp(-i b X)."""
    return np.array([[math.cos(b), -1j * math.sin(b)], [-1j * math.sin(b), math.cos(b)]], dtype=np.complex128)


def depolarizing1(p: float):
    """A0 = sqrt(1-3p/4) I, A1..3 = sqrt(p/4) {X,Y,Z}: Bloch vector shrinks by 1-p."""
    return (math.sqrt(1 - 3 * p / 4) * I2, math.sqrt(p / 4) * X, math.sqrt(p / 4) * Y, math.sqrt(p / 4) * Z)


def depolarizing2(p: float):
    """rho -> (1-p) rho + p I/4: A0 = sqrt(1-15p/16) I(x)I, others sqrt(p/16) P(x)Q."""
    out = []
    for a in "IXYZ":
        for b in "IXYZ":
            w = (1 - 15 * p / 16) if (a == "I" and b == "I") else p / 16
            out.append(math.sqrt(w) * np.kron(PAULI[a], PAULI[b]))
    return tuple(out)


def amplitude_damping(g: float):
    return (np.array([[1, 0], [0, math.sqrt(1 - g)]], dtype=np.complex128),
            np.array([[0, math.sqrt(g)], [0, 0]], dtype=np.complex128))


def dephasing(p: float):
    return (math.sqrt(1 - p) * I2, math.sqrt(p) * Z)


def random_unitary(rng: np.random.Generator, d: int) -> np.ndarray:
    """Haar-ish random unitary via QR of a complex Gaussian matrix (input only)."""
    A = rng.normal(size=(d, d)) + 1j * rng.normal(size=(d, d))
    Q, R = np.linalg.qr(A)
    return Q * (np.diag(R) / np.abs(np.diag(R)))


# ---------------------------------------------------------------------------
# small circuits (closed-form pins)
# ---------------------------------------------------------------------------


def bell() -> OpList:
    return OpList(2).gate(H, 0, name="H").gate(CX, 0, 1, name="CX")


def ghz(n: int) -> OpList:
    c = OpList(n).gate(H, 0, name="H")
    for q in range(1, n):
        c.gate(CX, 0, q, name="CX")
    return c


def cat_state(n: int = 60) -> OpList:
    """The paper's Fig. tnqvm_wave_fn_slice circuit: H(q0); CX(q0, qi) i=1..n-1."""
    return ghz(n)


def qft_into(c: OpList, qubits) -> OpList:
    """Textbook QFT with final swaps (qubit qubits[0] is the MSB)."""
    n = len(qubits)
    for j in range(n):
        c.gate(H, qubits[j], name="H")
        for k in range(j + 1, n):
            c.gate(cphase(2 * math.pi / 2 ** (k - j + 1)), qubits[k], qubits[j], name="CP")
    for j in range(n // 2):
        c.gate(SWAP, qubits[j], qubits[n - 1 - j], name="SWAP")
    return c


def ghz_qft(n: int = 8) -> OpList:
    """BASELINE config 1: GHZ_n then QFT_n; a_k = (1 + e^{-2 pi i k/N}) / sqrt(2N)."""
    return qft_into(ghz(n), list(range(n)))


def basis_qft(n: int, x: int) -> OpList:
    c = OpList(n)
    for q in range(n):
        if (x >> (n - 1 - q)) & 1:
            c.gate(X, q, name="X")
    return qft_into(c, list(range(n)))


def random_circuit(n: int, depth: int, seed: int, p2: float = 0.5) -> OpList:
    """Random brick circuit with Haar 1q/2q gates on random pairs (test input)."""
    rng = np.random.default_rng(seed)
    c = OpList(n)
    for _ in range(depth):
        perm = rng.permutation(n)
        for i in range(0, n - 1, 2):
            a, b = int(perm[i]), int(perm[i + 1])
            if rng.random() < p2:
                c.gate(random_unitary(rng, 4), a, b, name="U2")
            else:
                c.gate(random_unitary(rng, 2), a, name="U1")
    return c


# ---------------------------------------------------------------------------
# Sycamore-53 synthetic random circuits (paper P:L443-467)
# ---------------------------------------------------------------------------

SYCAMORE_ROWS = (
    "-----AB---",
    "----ABCD--",
    "---ABCDEF-",
    "--ABCDEFGH",
    "-ABCDEFGHI",
    "ABCDEFGHI-",
    "-CDEFGHI--",
    "--EFGHI---",
    "---GHI----",
    "----I-----",
)
SYCAMORE_DROPPED = ((3, 2),)
PATTERN_SEQ = "ABCDCDAB"


def grid_sites(rows, dropped=()):
    sites = []
    for r, line in enumerate(rows):
        for c, ch in enumerate(line):
            if ch != "-" and (r, c) not in dropped:
                sites.append((r, c))
    return sites  # row-major by (row, col)


def rect_sites(nrows: int, ncols: int):
    return [(r, c) for r in range(nrows) for c in range(ncols)]


def coupler_patterns(sites):
    """A/B (vertical) and C/D (horizontal) matchings; SURVEY §8(d)."""
    index = {s: i for i, s in enumerate(sites)}
    pats = {"A": [], "B": [], "C": [], "D": []}
    for (r, c), i in index.items():
        if (r + 1, c) in index:  # vertical pair, key r - c
            key = r - c
            if (key - 0) % 2 == 0:
                pats["A"].append((i, index[(r + 1, c)]))
            if (key - 1) % 2 == 0:
                pats["B"].append((i, index[(r + 1, c)]))
        if (r, c + 1) in index:  # horizontal pair, key c - r
            key = c - r
            if (key - 1) % 2 == 0:
                pats["C"].append((i, index[(r, c + 1)]))
            if (key - 0) % 2 == 0:
                pats["D"].append((i, index[(r, c + 1)]))
    for k in pats:
        pats[k].sort()
    return pats


def random_grid_circuit(sites, cycles: int, seed: int, theta=math.pi / 2, phi=math.pi / 6) -> OpList:
    """Sycamore-style RQC: per cycle a 1q layer from {sqrtX, sqrtY, sqrtW} (never the
    qubit's previous choice; the first layer uniform over all three), then fSim on
    pattern "ABCDCDAB"[c mod 8]; then a final 1q layer.  RNG call order: one
    ``rng.integers`` per qubit per layer, qubits in index order."""
    rng = np.random.default_rng(seed)
    n = len(sites)
    pats = coupler_patterns(sites)
    U2 = fsim(theta, phi)
    c = OpList(n)
    prev = [-1] * n

    def layer_1q():
        for q in range(n):
            if prev[q] < 0:
                g = int(rng.integers(3))
            else:
                choices = [j for j in range(3) if j != prev[q]]
                g = choices[int(rng.integers(2))]
            prev[q] = g
            c.gate(SYC_1Q[g], q, name=SYC_1Q_NAMES[g])

    for cyc in range(cycles):
        layer_1q()
        for (a, b) in pats[PATTERN_SEQ[cyc % 8]]:
            c.gate(U2, a, b, name="fSim")
    layer_1q()
    return c


def sycamore53(cycles: int, seed: int = 0) -> OpList:
    return random_grid_circuit(grid_sites(SYCAMORE_ROWS, SYCAMORE_DROPPED), cycles, seed)


def grid_rqc(nrows: int, ncols: int, cycles: int, seed: int = 0) -> OpList:
    return random_grid_circuit(rect_sites(nrows, ncols), cycles, seed)


def random_bitstring(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, 2, size=n).astype(np.int8)


# ---------------------------------------------------------------------------
# noisy grid circuit (BASELINE config 5)
# ---------------------------------------------------------------------------


def noisy_grid_circuit(nrows=4, ncols=5, cycles=8, seed=0, p1=1e-3, gamma=2e-3, p2=1e-2) -> OpList:
    """After each gate every touched qubit gets depolarizing(p1) then amplitude
    damping(gamma); each fSim is followed (before those) by a 2q depolarizing(p2)."""
    base = grid_rqc(nrows, ncols, cycles, seed)
    c = OpList(base.nq)
    D1, AD, D2 = depolarizing1(p1), amplitude_damping(gamma), depolarizing2(p2)
    for op in base.ops:
        c.ops.append(op)
        if len(op.qubits) == 2:
            c.kraus(D2, *op.qubits, name="dep2")
        for q in op.qubits:
            c.kraus(D1, q, name="dep1")
            c.kraus(AD, q, name="ad")
    return c


# ---------------------------------------------------------------------------
# QAOA MaxCut (BASELINE config 4)
# ---------------------------------------------------------------------------


def regular_graph(d: int, n: int, seed: int):
    import networkx as nx
    g = nx.random_regular_graph(d, n, seed=seed)
    return sorted(tuple(sorted(e)) for e in g.edges())


def qaoa_circuit(n: int, edges, gammas, betas) -> OpList:
    """H^{(x)n}; per layer prod_E exp(-i g Z_u Z_v), then prod_q exp(-i b X_q)."""
    c = OpList(n)
    for q in range(n):
        c.gate(H, q, name="H")
    for g, b in zip(gammas, betas):
        for (u, v) in edges:
            c.gate(rzz(g), u, v, name="RZZ")
        for q in range(n):
            c.gate(rx(b), q, name="RX")
    return c


def maxcut_terms(edges):
    """H = sum_E Z_u Z_v (coefficient 1): list of (coeff, [(q, 'Z'), ...])."""
    return [(1.0, [(u, "Z"), (v, "Z")]) for (u, v) in edges]


QAOA_GAMMAS = (0.2, 0.4)
QAOA_BETAS = (0.6, 0.3)


def qaoa40(seed: int = 0):
    edges = regular_graph(3, 40, seed)
    return qaoa_circuit(40, edges, QAOA_GAMMAS, QAOA_BETAS), maxcut_terms(edges)
